// capi.cpp -- C ABI (include/safekv_b200.h): rule snapshots, context lifetime, and the
// host orchestration of the device stages of one admission batch.  Host code only
// sequences kernels and moves buffers; every per-token / per-block / per-entry
// computation runs on the device (kernels.cu).  There is no CPU fallback path.
#include <cuda_runtime.h>

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "../../include/safekv_b200.h"
#include "ctx.hpp"
#include "rules.hpp"

struct skv_rules {
  skv::RuleSetSpec spec;
  skv::DfaTables dfa;       // the whole rule set's automaton (skv_rules_dfa; the rule order)
  skv::RuleGroups groups;   // the device's automata: consecutive groups of <= 16 enabled rules
  std::vector<uint32_t> enabled;  // rule-list position of the j-th enabled rule (mask bit j)
  bool whole = false;             // dfa holds the whole set (<= 32 enabled rules: one u32 mask)
};

#ifndef SKV_COMMIT_FLAT_HOST
#define SKV_COMMIT_FLAT_HOST 0  // set with SKV_COMMIT_FLAT: the flat commit needs bprompt from the probe
#endif
#ifndef SKV_REC_BESIDE
#define SKV_REC_BESIDE 0  // measured: 0.82 ms beside vs 0.72 fused (DESIGN 5.3)
#endif
constexpr bool kRecordBeside = SKV_REC_BESIDE != 0;
constexpr size_t kEpochEvPre = 128;  // events read back with an epoch's count
constexpr int kEpochCountSlot = 56;  // host_small word of the epoch's event count
constexpr uint64_t kEpochSplitMin = 65536;  // touched entries from which the epoch runs as six kernels
#ifndef SKV_STREAM_PRIO
#define SKV_STREAM_PRIO 0
#endif
#ifndef SKV_PF_CHAIN
#define SKV_PF_CHAIN 1
#endif
constexpr bool kPrefetchChain = SKV_PF_CHAIN != 0 && !SKV_COMMIT_FLAT_HOST;

namespace {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StateError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CapacityError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ArgError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) ck((x), #x)

// every host sync point also surfaces launch failures (bad config, smem opt-in, ...)
void sync_check(cudaStream_t s) {
  ck(cudaGetLastError(), "kernel launch");
  ck(cudaStreamSynchronize(s), "stream synchronize");
  ck(cudaGetLastError(), "kernel execution");
}

template <typename T>
T* dalloc(size_t n, std::vector<void*>& owned) {
  void* p = nullptr;
  if (n == 0) n = 1;
  CK(cudaMalloc(&p, n * sizeof(T)));
  owned.push_back(p);
  return static_cast<T*>(p);
}

uint64_t next_pow2(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

int log2u(uint64_t x) {
  int b = 0;
  while ((1ull << b) < x) ++b;
  return b;
}

bool getenv_flag(const char* name) {
  const char* v = std::getenv(name);
  return v && *v && *v != '0';
}

uint64_t fnv_u32_host(uint64_t h, uint32_t v) {
  for (int i = 0; i < 4; ++i) h = (h ^ ((v >> (8 * i)) & 0xff)) * 0x100000001b3ULL;
  return h;
}

}  // namespace

struct skv_ctx {
  skv_config cfg{};
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  std::vector<void*> owned;

  // rules
  skv_rules rules_host;
  // one device automaton per rule group (skv_rules::groups): the general kernel's tables and,
  // for B = 16 / W = 32, k_hash_scan16's
  struct DevGroup {
    skv::DevRules dev{};
    void* buf = nullptr;
    skv::DevRules16 r16{};
    skv::HSLayout layout{};
    uint32_t smem = 0, shift = 0, word = 0;  // mask bits: word `word`, from bit `shift`
    int grid = 0;
  };
  std::vector<DevGroup> groups;
  uint32_t mask_words = 1;      // words of the active rule set's window masks
  uint32_t mask_words_cap = 1;  // words bmask / alt_bmask hold per block (max_blocks stride)
  bool rules_loaded = false;

  // index
  skv::Index ix;
  uint64_t entries = 0;

  // monitor window state
  skv::SetHdr* set_hdr = nullptr;
  ulonglong2* set_tab = nullptr;
  uint32_t* replay = nullptr;      // entries needing an ordered monitor replay
  uint32_t rec_batch = 0;          // admit-batch id (monitor stamps)
  uint32_t wstart = 1;             // first batch id of the current monitor window
  uint32_t pool_cap = 0;
  uint32_t* touched[2] = {nullptr, nullptr};
  // [0]=pool_count [1..2]=n_touched[2] [3]=n_cands [4]=n_events [5]=err_flag [6]=n_batch
  // [7]=n_fix [8]=n_replay [9]=n_keys [10]=matched_total
  uint32_t* counters = nullptr;
  unsigned long long* n_new = nullptr;
  int cur = 0;
  uint32_t* cands = nullptr;
  uint32_t* fired = nullptr;
  void* events = nullptr;
  uint64_t epoch = 0;

  // batch buffers
  uint64_t max_prompts = 0, max_tokens = 0, max_blocks = 0;
  uint32_t* d_tokens = nullptr;
  uint8_t* d_tok8 = nullptr;  // byte-token staging (skv_batch::token_bytes)
  uint64_t* d_off = nullptr;
  uint64_t* d_users = nullptr;
  uint8_t* d_owners = nullptr;
  uint32_t* counts = nullptr;
  uint32_t* blk_off = nullptr;
  uint32_t* first_sens = nullptr;
  uint32_t* matched = nullptr;
  uint32_t* exist = nullptr;
  uint8_t* tier = nullptr;
  uint64_t* bh = nullptr;
  uint64_t* bd = nullptr;
  uint32_t* bmask = nullptr;
  uint8_t* blabel = nullptr;
  uint32_t* bprompt = nullptr;  // block -> prompt (written by the probe, read by the flat commit)
  // eviction (skv_enable_eviction): bookkeeping array + lazily allocated work buffers
  bool evict_on = false;
  bool evict_tiered = false;  // victims move HBM -> DRAM instead of leaving
  uint64_t tombstones = 0;  // evicted slots not re-inserted (they keep their slot)
  uint32_t* ev_counts = nullptr;
  uint32_t* ev_incl = nullptr;
  uint64_t node_next = 1;  // next_node_id_ (cache_index.hpp:832); the root is node 0
  void* ev_temp = nullptr;
  size_t ev_temp_bytes = 0;
  unsigned long long* ev_eff = nullptr;
  uint32_t* ev_n = nullptr;
  uint32_t* late = nullptr;     // commit: (child slot, parent block) links applied after the claims
  uint8_t* bdecision = nullptr;
  uint32_t* bslot = nullptr;
  uint8_t* bmeta = nullptr;    // per matched block: tier | creator == user << 2 (TTFT epilogue)
  uint32_t* plen = nullptr;    // tokens per prompt of the last admitted batch
  uint32_t* alt_plen = nullptr;
  double* d_ttft = nullptr;    // skv_admit_ttft scratch
  uint32_t* d_intra = nullptr;
  uint32_t* d_inter = nullptr;
  uint64_t* d_reqid = nullptr;
  skv::CostModelDev cost{};
  uint64_t admitted_prompts = 0;  // request ids of the last batch default to [admitted_prompts - N, ...)
  uint32_t last_n = 0;            // prompts of the last skv_admit
  unsigned long long *keys_a = nullptr, *keys_b = nullptr;  // ordered-replay access keys
  uint32_t* fix_list = nullptr;  // commit: duplicate-key slots, depths, prompts, late children (4 x max_blocks)
  skv::UserTable users_tab{};     // interned UserIds (Rec::creator)
  uint32_t* uidx = nullptr;       // interned user of every prompt of the last admit
  void* temp = nullptr;
  size_t temp_bytes = 0;
  uint32_t* host_small = nullptr;  // pinned scratch for small readbacks
  skv_event* host_events = nullptr;  // pinned: the first kEpochEvPre events of an epoch, read with its count
  uint32_t* hs_map = nullptr;      // block -> prompt of a short-prompt batch (stages 1-2 on the context stream)
  uint32_t* alt_hs_map = nullptr;  // ... of a prefetched batch (side stream)
  int n_sm = 148;
  uint32_t rec_grid = 0;

  // set when a failed call left device state that no longer follows the reference (every
  // later batch call raises StateError with this reason; export still works)
  std::string poisoned;
  std::vector<skv_event> last_events;  // every event of the last skv_epoch, sorted by key
  // replicated layer (skv_set_replicated_depth): device scratch of the export / apply
  bool rep_sync_due = false;  // a committed batch waits for skv_replica_export / apply
  skv_rep_entry* rep_ents = nullptr;   // export scratch (new_cap)
  skv_rep_access* rep_accs = nullptr;  // export scratch (pair capacity)
  uint64_t* rep_gids = nullptr;        // per prompt of the last batch
  void* rep_in = nullptr;              // apply input (grown on demand)
  size_t rep_in_bytes = 0;
  uint32_t* rep_slots = nullptr;
  uint32_t* rep_uidx = nullptr;
  skv::RepScratch rep_w;  // device merge of the ranks' access exports
  size_t rep_in_ents = 0;
  // pending batch (between admit and commit)
  bool pending = false;
  bool dropped_by_evict = false;  // the last admitted batch was dropped by skv_evict
  bool no_record = false;         // skv_lookup / skv_insert: the admit records no accesses
  // monitor records of the last admit, executed inside the commit kernel (overlapping
  // the claims), or on their own when the batch is not committed
  bool rec_pending = false;
  bool pending_labels = false;  // skv_set_label_policy: new entries start PendingPrivate
  bool adm_lazy = false;  // the last admit's readbacks are pending (resolve_admit)
  bool adm_use_pf = false;
  uint32_t adm_launched = 0;
  skv::MonCtx rec_mon{};
  const uint64_t* rec_users = nullptr;
  uint32_t rec_n = 0;
  uint32_t p_n = 0;
  uint64_t p_blocks = 0;
  const uint64_t* p_users = nullptr;
  const uint8_t* p_owners = nullptr;
  uint32_t batch_id = 0;

  cudaEvent_t ev[10] = {};  // 0-4 admit, 5-6 commit, 8-9 epoch
  skv_stage_times times{};

  // cross-batch pipelining (skv_prefetch): stages 1-2 of the next batch on a side stream
  // into the alternate buffer set {counts, blk_off, first_sens, bd, bmask}
  cudaStream_t side = nullptr;
  cudaStream_t rec_stream = nullptr;  // a batch's monitor records, beside its commit
  cudaEvent_t rec_start = nullptr, rec_done = nullptr;
  cudaEvent_t pf_done = nullptr;
  uint32_t *alt_counts = nullptr, *alt_blk_off = nullptr, *alt_first_sens = nullptr, *alt_bmask = nullptr;
  // the prefetched batch's chained keys, labels and slot init (k_chain on the side stream)
  uint64_t* alt_bh = nullptr;
  uint8_t* alt_blabel = nullptr;
  uint32_t* alt_bslot = nullptr;
  uint64_t* alt_bd = nullptr;
  bool pf_valid = false;
  // bracket a prefetched hash/scan (side stream); two pairs, alternating, so that the admit
  // consuming prefetch k still reads its own pair after prefetch k+1 has been enqueued
  cudaEvent_t pf_ev[2][2] = {};
  int pf_pair = 0;      // pair of the staged prefetch
  int adm_pf_pair = 0;  // pair of the prefetch the last admit consumed
  void* side_temp = nullptr;
  size_t side_temp_bytes = 0;
  bool pf_on_device = false;
  const void* pf_tokens = nullptr;
  const void* pf_offsets = nullptr;
  const void* pf_users = nullptr;
  const void* pf_owners = nullptr;
  // host-batch staging set (skv_prefetch of a host batch copies into it on the side stream)
  uint32_t* alt_tokens = nullptr;
  uint8_t* alt_tok8 = nullptr;  // byte-token staging (skv_batch::token_bytes)
  uint64_t* alt_off = nullptr;
  uint64_t* alt_users = nullptr;
  uint8_t* alt_owners = nullptr;
  uint32_t pf_n = 0;
  uint64_t pf_ntok = 0;

  // host-input staging ring (skv_stage): a host batch's H2D into one of two device slots on
  // a copy stream, ahead of its prefetch / admit, so the copy of batch k+1 runs while batch k
  // is admitted and committed (the PCIe copy is the end-to-end bottleneck).  A slot is FREE,
  // STAGED (copy queued), PREFETCHED (stages 1-2 queued on it) or INUSE (its users / owners
  // are read until the batch's commit); free_ev orders the next copy after the last reader.
  enum SlotState { kSlotFree, kSlotStaged, kSlotPrefetched, kSlotInUse };
  struct HostSlot {
    uint32_t* tok = nullptr;
    uint8_t* tok8 = nullptr;
    uint64_t* off = nullptr;
    uint64_t* users = nullptr;
    uint8_t* owners = nullptr;
    cudaEvent_t ready = nullptr, free_ev = nullptr;
    SlotState state = kSlotFree;
    const void* id_tok = nullptr;
    const uint64_t* id_off = nullptr;
    const uint64_t* id_users = nullptr;
    const uint8_t* id_owners = nullptr;
    uint32_t n = 0;
    uint64_t ntok = 0;
    bool bytes = false;
  };
  static constexpr int kHostSlots = 3;  // batch k in use, k+1 prefetched, k+2 copying: the copy engine never waits
  HostSlot hslot[kHostSlots];
  cudaStream_t copy = nullptr;

  // A.9 tier budgets (skv_set_tier_budget): capacities and used blocks per tier; the commit then
  // makes room for each insert (kernels.cu "A.9")
  bool budget_on = false;
  uint64_t bud_cap[3] = {0, 0, 0}, bud_used[3] = {0, 0, 0};
  uint32_t* vstamp = nullptr;  // per slot: 0 pinned, p + 1 first walking prompt, ~0 none
  uint32_t* mark_list = nullptr;
  uint32_t* n_mark = nullptr;
  uint32_t mark_cap = 0;
  ulonglong2* dry_tab = nullptr;
  uint32_t* dry_minp = nullptr;
  uint64_t dry_cap = 0;
  uint32_t* dry_slot = nullptr;
  uint32_t* needed = nullptr;
  skv::BudgetSim* sim = nullptr;
  unsigned long long* nb_dev = nullptr;
  std::vector<uint32_t> dropped;  // prompts of the last commit whose insert could not make room
  int pf_slot = -1;   // slot of the prefetched batch

  // CUDA graphs for small batches (a device-resident batch admitted without per-block outputs,
  // no eviction / budgets / replicated layer / pending prefetch): each phase's launches are
  // captured once per buffer set and replayed with one cudaGraphLaunch; the per-step scalars the
  // kernels need (batch and window stamps, current window list, epoch) come from the device step
  // state dstate = {batch, wstart, cur, stamp, epoch lo, epoch hi}, copied from pinned host
  // memory before each launch (one slot per phase).  A small batch's step is otherwise bound by
  // host issue: ~40 API calls for ~80 us of kernels (config 1).
  struct GraphCache {  // the last few instantiated graphs of a phase, by key (most recent first)
    struct Item {
      cudaGraphExec_t exec = nullptr;
      std::vector<uintptr_t> key;
    };
    std::vector<Item> items;
  };
  GraphCache g_admit, g_commit, g_epoch;
  bool graphs = true;
  bool capturing = false;
  bool adm_graph = false;    // the pending batch was admitted through its graph
  bool adm_nb_dev = false;   // the pending batch's block count arrives in host_small[20]
  double probe_est = -1.0;   // mean matched blocks per prompt of the last resolved admit (probe wave split)
  uint64_t touched_est = 0;  // entries in the current window list after the last commit (epoch shape)
  bool lazy_outputs = false; // skv_step: the admit's output copies complete with the step's synchronisation
  skv_admit_out* adm_out = nullptr;  // ... whose summary resolve_admit fills
  uint32_t* dstate = nullptr;
  uint32_t* hstate = nullptr;  // pinned, 3 x 8 words (admit, commit, epoch)
  uint64_t rules_gen = 0;      // bumped by upload_rules (the admit graph bakes the rule tables in)
  int use_slot = -1;  // slot of the pending (admitted) batch
};

namespace {

thread_local std::string g_create_err;

int fail(skv_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

template <typename F>
int guard(skv_ctx* c, F&& f) {
  try {
    return f();
  } catch (const skv::ParseError& e) {
    return fail(c, SKV_ERR_PARSE, e.what());
  } catch (const skv::CompileError& e) {
    return fail(c, SKV_ERR_COMPILE, e.what());
  } catch (const skv::ConfigError& e) {
    return fail(c, SKV_ERR_CONFIG, e.what());
  } catch (const CudaError& e) {
    return fail(c, SKV_ERR_CUDA, e.what());
  } catch (const StateError& e) {
    return fail(c, SKV_ERR_STATE, e.what());
  } catch (const CapacityError& e) {
    return fail(c, SKV_ERR_CAPACITY, e.what());
  } catch (const ArgError& e) {
    return fail(c, SKV_ERR_ARG, e.what());
  } catch (const std::exception& e) {
    return fail(c, SKV_ERR_INTERNAL, e.what());
  }
}

// Whether a group automaton fits the general kernel's device tables (u16 row offsets below the
// 32 KB copy region, <= 63 byte classes, u16 copy-row rule masks: <= 16 rules per group).
uint32_t mask_words_of(const skv_rules& r) {
  return std::max<uint32_t>(1, static_cast<uint32_t>((r.enabled.size() + 31) / 32));
}

bool fits_device(const skv::DfaTables& d) {
  const uint32_t C = d.n_classes, S = d.n_states, row = (C + 1) * 2;
  if (C + 1 > 64 || d.rule_index.size() > 16) return false;
  if (((S * row + 15) & ~15u) > skv::kAccRegion) return false;
  std::set<std::pair<uint32_t, uint32_t>> copies;
  for (uint32_t s = 0; s < S; ++s)
    for (uint32_t k = 0; k <= C; ++k)
      if (d.acc[s * (C + 1) + k]) copies.emplace(k < C ? d.next[s * C + k] : UINT32_MAX, d.acc[s * (C + 1) + k]);
  return skv::kAccRegion + copies.size() * row <= 65535;
}

void free_group(skv_ctx::DevGroup& g) {
  for (void* p : {g.buf, static_cast<void*>(g.r16.img), static_cast<void*>(g.r16.hi), static_cast<void*>(g.r16.full)})
    if (p) cudaFree(p);
  g = skv_ctx::DevGroup{};
}

// Device form of one group's DFA (see ctx.hpp DevRules): rows at the top of the 32 KB region,
// accepting transitions pointing at copies of their target row above it.
void build_group(skv_ctx* c, const skv::DfaTables& d, skv_ctx::DevGroup& g) {
  const uint32_t C = d.n_classes, S = d.n_states, row = (C + 1) * 2;
  const uint32_t norm = S * row;
  if (!fits_device(d)) throw skv::CompileError("device DFA: a rule group exceeds the device tables");
  // accepting transitions -> copies of the target row in the region above 32 KB
  std::map<std::pair<uint32_t, uint32_t>, uint32_t> copy_of;  // (target, acc) -> copy index
  std::vector<std::pair<uint32_t, uint32_t>> copies;
  auto copy_index = [&](uint32_t target, uint32_t acc) {
    auto it = copy_of.emplace(std::make_pair(target, acc), static_cast<uint32_t>(copies.size()));
    if (it.second) copies.emplace_back(target, acc);
    return it.first->second;
  };
  // rows are placed at the top of the 32 KB region, [row_base, 32768), so that the
  // SMEM-resident part [row_base, fast_bytes) is contiguous (no gap before the copies)
  const uint32_t row_base = skv::kAccRegion - ((norm + 15) & ~15u);
  std::vector<uint16_t> entry(static_cast<size_t>(S) * (C + 1), 0);
  std::vector<uint32_t> full(static_cast<size_t>(S) * (C + 1), 0);
  for (uint32_t s = 0; s < S; ++s) {
    for (uint32_t k = 0; k <= C; ++k) {
      uint32_t acc = d.acc[s * (C + 1) + k];
      uint32_t t = k < C ? d.next[s * C + k] : 0;
      uint32_t fast = k < C ? row_base + t * row : 0;
      if (acc) fast = skv::kAccRegion + copy_index(k < C ? t : UINT32_MAX, acc) * row;
      entry[s * (C + 1) + k] = static_cast<uint16_t>(fast);
      full[s * (C + 1) + k] = (acc << 16) | (k < C ? row_base + t * row : 0);
    }
  }
  const uint32_t fast_bytes = skv::kAccRegion + static_cast<uint32_t>(copies.size()) * row;
  std::vector<uint8_t> fast(fast_bytes, 0);
  std::memcpy(fast.data() + row_base, entry.data(), entry.size() * 2);
  for (size_t j = 0; j < copies.size(); ++j)
    if (copies[j].first != UINT32_MAX)  // EOS pseudo rows carry no transitions
      std::memcpy(fast.data() + skv::kAccRegion + j * row, entry.data() + copies[j].first * (C + 1), row);
  uint8_t class2[256];
  for (int b = 0; b < 256; ++b) class2[b] = static_cast<uint8_t>(d.class_map[b] * 2);
  std::vector<uint16_t> copy_acc(copies.size() + 1, 0);
  for (size_t j = 0; j < copies.size(); ++j) copy_acc[j] = static_cast<uint16_t>(copies[j].second);
  const uint32_t inv = static_cast<uint32_t>(((1ull << 32) + row - 1) / row);
  for (uint32_t j = 0; j < copies.size(); ++j)  // exactness of the reciprocal on every copy offset
    if (static_cast<uint32_t>((static_cast<uint64_t>(j * row) * inv) >> 32) != j)
      throw skv::CompileError("device DFA: copy-row reciprocal not exact");
  const size_t fast_al = (fast_bytes + 15) & ~size_t(15);
  const size_t full_bytes = full.size() * 4;
  const size_t acc_bytes = copy_acc.size() * 2;
  CK(cudaMalloc(&g.buf, fast_al + full_bytes + 256 + acc_bytes + 64));
  uint8_t* base = static_cast<uint8_t*>(g.buf);
  CK(cudaMemcpyAsync(base, fast.data(), fast_bytes, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(base + fast_al, full.data(), full_bytes, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(base + fast_al + full_bytes, class2, 256, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(base + fast_al + full_bytes + 256, copy_acc.data(), acc_bytes, cudaMemcpyHostToDevice,
                     c->stream));
  skv::DevRules& R = g.dev;
  R.copy_acc = reinterpret_cast<uint16_t*>(base + fast_al + full_bytes + 256);
  R.n_copies = static_cast<uint32_t>(copies.size());
  R.copy_inv = inv;
  R.fast = reinterpret_cast<uint16_t*>(base);
  R.full = reinterpret_cast<uint32_t*>(base + fast_al);
  R.class2 = base + fast_al + full_bytes;
  R.fast_bytes = fast_bytes;
  R.norm_bytes = norm;
  R.row_bytes = row;
  R.start_row = row_base + d.start * row;
  R.row_base = row_base;
  R.eos2 = C * 2;
  R.n_enabled = static_cast<uint32_t>(d.rule_index.size());
  g.layout = skv::hash_scan_layout(R, c->cfg.block_tokens, c->cfg.window_tokens);
  g.smem = g.layout.total;
  if (g.layout.warps == 0 || g.smem > 227 * 1024)
    throw skv::ConfigError("hash/scan shared-memory footprint exceeds 227 KB (block_tokens too large)");
  g.grid = skv::hash_scan_grid(c->device, g.smem, 32 * g.layout.warps);
  if (g.grid <= 0) throw CudaError("k_hash_scan: shared-memory opt-in / occupancy query failed");
}

// The B = 16 / W = 32 automaton of k_hash_scan16 (ctx.hpp DevRules16, hash_scan16.cuh): column t
// < 128 of the image holds, for every state index (S base states, then their S shadow copies),
// v(next) = 2 * index of the next state -- the shadow copy when the transition accepts a rule
// or the state is a shadow already; column 128 holds the end-of-text rule mask.  Not built
// (the general kernel runs) for other shapes or when the image does not fit SMEM beside the
// per-warp task queues.
void build_group16(skv_ctx* c, const skv::DfaTables& d, skv_ctx::DevGroup& g) {
  skv::DevRules16& R = g.r16;
  const uint32_t S = d.n_states, C = d.n_classes;
  if (c->cfg.block_tokens != 16 || c->cfg.window_tokens != 32 || 4ull * S >= 65536) return;
  const uint32_t S2 = 2 * S, colbytes = 4 * S;
  const uint32_t img_bytes = 129 * colbytes;
  uint32_t q_cap = 256;  // deferred tasks per warp: shrink to fit, at least 3 segments x 32 lanes
  constexpr uint32_t kSmemMax = 227 * 1024 - 1024;  // the kernel's static shared (image mbarrier) beside it
  while (q_cap > 96 && skv::hash_scan16_smem(img_bytes, q_cap) > kSmemMax) q_cap -= 32;
  if (skv::hash_scan16_smem(img_bytes, q_cap) > kSmemMax) return;
  std::vector<uint16_t> img(129ull * S2 + 8, 0), hi(128ull * S2, 0);
  std::vector<uint32_t> full(256ull * S, 0);
  for (uint32_t b = 0; b < 256; ++b) {
    const uint32_t k = d.class_map[b];
    uint16_t* col = b < 128 ? &img[static_cast<size_t>(b) * S2] : &hi[static_cast<size_t>(b - 128) * S2];
    for (uint32_t s = 0; s < S; ++s) {
      const uint32_t t = d.next[s * C + k], acc = d.acc[s * (C + 1) + k];
      col[s] = static_cast<uint16_t>(2 * (t + (acc ? S : 0)));
      col[S + s] = static_cast<uint16_t>(2 * (t + S));
      full[static_cast<size_t>(b) * S + s] = (acc << 16) | (2 * t);
    }
  }
  for (uint32_t s = 0; s < S; ++s)
    img[128ull * S2 + s] = img[128ull * S2 + S + s] = static_cast<uint16_t>(d.acc[s * (C + 1) + C]);
  const uint32_t smem = skv::hash_scan16_smem(img_bytes, q_cap);
  const int grid = skv::hash_scan16_grid(c->device, smem);
  if (grid <= 0) return;
  const size_t img_al = (img_bytes + 15) & ~size_t(15);
  CK(cudaMalloc(&R.img, img_al));
  CK(cudaMalloc(&R.hi, hi.size() * 2));
  CK(cudaMalloc(&R.full, full.size() * 4));
  CK(cudaMemcpyAsync(R.img, img.data(), img_al, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(R.hi, hi.data(), hi.size() * 2, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(R.full, full.data(), full.size() * 4, cudaMemcpyHostToDevice, c->stream));
  R.img_bytes = img_bytes;
  R.colbytes = colbytes;
  R.s2 = S2;
  R.v_start = 2 * d.start;
  R.q_cap = q_cap;
  R.smem = smem;
  R.grid = grid;
  R.ok = true;
}

// The rule set's device automata (one per rule group); replaces the previous set atomically
// (RuleEngine::load_rules swap, detection.hpp:238-241) once every table is on the device.
void upload_rules(skv_ctx* c, const skv_rules& r) {
  std::vector<skv_ctx::DevGroup> gs(r.groups.groups.size());
  try {
    for (size_t i = 0; i < gs.size(); ++i) {
      build_group(c, r.groups.groups[i], gs[i]);
      build_group16(c, r.groups.groups[i], gs[i]);
      gs[i].shift = r.groups.first_bit[i] % 32;
      gs[i].word = r.groups.first_bit[i] / 32;
    }
    sync_check(c->stream);
    const uint32_t words = mask_words_of(r);
    if (words > c->mask_words_cap) {  // a wider rule library: window masks of `words` words per block
      if (c->side) CK(cudaStreamSynchronize(c->side));
      const uint64_t NB = std::max<uint64_t>(c->max_blocks, 1);
      uint32_t* nb = nullptr;
      uint32_t* na = nullptr;
      CK(cudaMalloc(&nb, NB * words * 4));
      if (cudaMalloc(&na, NB * words * 4) != cudaSuccess) {
        cudaFree(nb);
        throw CudaError("cudaMalloc: rule mask words");
      }
      for (auto& p : c->owned)
        if (p == c->bmask || p == c->alt_bmask) {
          cudaFree(p);
          p = p == c->bmask ? static_cast<void*>(nb) : static_cast<void*>(na);
        }
      c->bmask = nb;
      c->alt_bmask = na;
      c->mask_words_cap = words;
    }
    c->mask_words = words;
  } catch (...) {
    for (auto& g : gs) free_group(g);
    throw;
  }
  for (auto& g : c->groups) free_group(g);
  c->groups = std::move(gs);
  c->rules_host = r;
  c->rules_loaded = true;
  ++c->rules_gen;
}

skv::MonCtx monitor_ctx(skv_ctx* c) {
  skv::MonCtx m;
  m.hdr = c->set_hdr;
  m.tab = c->set_tab;
  m.pool_cap = c->pool_cap;
  m.pool_count = c->counters + 0;
  m.touched = c->touched[c->cur];
  m.n_touched = c->counters + 1 + c->cur;
  m.batch = ++c->rec_batch;
  m.wstart = c->wstart;
  m.err = c->counters + 5;
  m.matched_total = c->counters + 10;
  return m;
}

// Stages 1+2 on stream `st`: digests, window rule masks and first sensitive block of a
// batch whose block offsets are already in blk_off (the kernel reads the block count
// from blk_off[N], so no host round trip is needed).
void stage12(skv_ctx* c, cudaStream_t st, const uint32_t* tokens, const uint64_t* off, uint32_t N, uint64_t n_tokens,
             uint64_t nb_hint, uint32_t* blk_off, uint32_t* first_sens, uint64_t* bd, uint32_t* bmask,
             bool overlapped = false) {
  static const bool force_general = getenv_flag("SKV_HS_GENERAL");
  static const bool pf_general = getenv_flag("SKV_PF_GENERAL");
  // a prefetch (stages 1-2 of the next batch beside the current commit) runs on a quarter of the
  // SMs: the one-CTA-per-SM kernel would otherwise hold every SM until it ends and serialise the
  // commit behind it (measured: 1.13 ms per config-2 step at full grid, 0.97 at a quarter)
  static const int pf_frac = getenv("SKV_H16_PF_FRAC") ? atoi(getenv("SKV_H16_PF_FRAC")) : 4;
  static const int pf_warps = getenv("SKV_H16_PF_WARPS") ? atoi(getenv("SKV_H16_PF_WARPS")) : 8;
  const uint64_t NB = std::max<uint64_t>(c->max_blocks, 1);
  if (c->mask_words > 1) {  // words >= 1 are only OR-ed into by their groups
    const uint64_t nb = std::min<uint64_t>(NB, std::max<uint64_t>(nb_hint, n_tokens / c->cfg.block_tokens));
    for (uint32_t w = 1; w < c->mask_words; ++w) CK(cudaMemsetAsync(bmask + w * NB, 0, nb * 4, st));
  }
  // one pass per rule group: the first stores the digests and the window masks, the others OR
  // their masks in at their rules' bits (a rule set larger than one device automaton)
  for (size_t gi = 0; gi < c->groups.size(); ++gi) {
    const skv_ctx::DevGroup& g = c->groups[gi];
    if (g.r16.ok && !force_general && !(overlapped && pf_general)) {
      const skv::DevRules16& R = g.r16;
      skv::HS16Args h;
      h.tokens = tokens;
      h.tok_off = off;
      h.blk_off = blk_off;
      h.n_prompts = N;
      h.n_tokens = n_tokens;
      h.digest_init = fnv_u32_host(0xcbf29ce484222325ULL, 16);
      h.img = R.img;
      h.img_bytes = R.img_bytes;
      h.hi = R.hi;
      h.full = R.full;
      h.colbytes = R.colbytes;
      h.s2 = R.s2;
      h.v_start = R.v_start;
      h.q_cap = R.q_cap;
      h.mask_shift = g.shift;
      h.first = gi == 0;
      h.d_out = bd;
      h.mask_out = bmask + g.word * NB;
      h.first_sens = first_sens;
      // a large batch: one 32-warp CTA per SM, a warp per 32-block chunk in turn.  A small batch
      // (fewer chunks than 32 warps x SMs): its chunks spread over the SMs with fewer warps per CTA
      // (the per-SM issue of 32 warps would otherwise bound it on a handful of SMs)
      const uint64_t nb_est = nb_hint ? nb_hint : n_tokens / 16;
      const uint64_t chunks = std::max<uint64_t>(1, (nb_est + 31) / 32);
      uint64_t grid = R.grid;
      int warps = 32;
      if (chunks < 32ull * R.grid) {
        warps = static_cast<int>(std::clamp<uint64_t>((chunks + R.grid - 1) / R.grid, 4, 32));
        grid = std::min<uint64_t>(R.grid, (chunks + warps - 1) / warps);
      }
      uint32_t smem = R.smem;
      if (overlapped && pf_warps > 0 && warps == 32) {
        // a prefetch beside the previous batch's commit: one small CTA on every SM, which fits next
        // to the commit's CTAs (registers / SMEM) and uses the issue slots its memory stalls leave
        warps = pf_warps;
        smem = skv::hash_scan16_smem(R.img_bytes, R.q_cap, static_cast<uint32_t>(pf_warps));
      } else if (overlapped && pf_frac > 1) {
        // ... or (SKV_H16_PF_WARPS=0) a quarter of the SMs with full CTAs
        grid = std::min<uint64_t>(grid, std::max<uint64_t>(1, R.grid / pf_frac));
      }
      // short prompts (< ~34 blocks): the chunk geometry comes from a block -> prompt map
      if (N && nb_est / N < 34) {
        uint32_t*& map = overlapped ? c->alt_hs_map : c->hs_map;
        if (!map) map = dalloc<uint32_t>(std::max<uint64_t>(c->max_blocks, 1), c->owned);
        skv::launch_block_prompts(blk_off, N, map, st);
        h.bmap = map;
      }
      skv::launch_hash_scan16(h, static_cast<int>(grid), smem, st, warps);
      continue;
    }
    skv::HashScanArgs a;
    a.tokens = tokens;
    a.tok_off = off;
    a.blk_off = blk_off;
    a.n_prompts = N;
    a.n_tokens = n_tokens;
    a.n_blocks = static_cast<uint32_t>(nb_hint);  // grid-size hint only; 0 = unknown
    a.B = c->cfg.block_tokens;
    a.W = c->cfg.window_tokens;
    a.digest_init = fnv_u32_host(0xcbf29ce484222325ULL, a.B);
    a.rules = g.dev;
    a.mask_shift = g.shift;
    a.first = gi == 0;
    a.d_out = bd;
    a.mask_out = bmask + g.word * NB;
    a.first_sens = first_sens;
    a.off_list = g.layout.off_list;
    a.stage = g.layout.stage;
    a.buf_gap = g.layout.buf_gap;
    a.n_gap = g.layout.n_gap;
    a.buf_tail = g.layout.buf_tail;
    skv::launch_hash_scan(a, g.grid, g.smem, 32 * g.layout.warps, st);
  }
}

// Offsets of a host batch: [0, n_tokens], non-decreasing.  Returns the block count.
uint64_t host_block_count(const skv_batch* b, uint32_t B) {
  const uint32_t N = b->n_prompts;
  if (b->offsets[0] != 0 || b->offsets[N] != b->n_tokens) throw ArgError("offsets must span [0, n_tokens]");
  uint64_t n_blocks = 0;
  for (uint32_t p = 0; p < N; ++p) {
    if (b->offsets[p + 1] < b->offsets[p]) throw ArgError("offsets must be non-decreasing");
    n_blocks += (b->offsets[p + 1] - b->offsets[p]) / B;
  }
  return n_blocks;
}

// CUDA-event interval; a failed query (an event never recorded, or recorded on another
// device) is reported as -1 rather than a stale or zero time
float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
    cudaGetLastError();
    return -1.0f;
  }
  return ms;
}

// NVTX range of a C-ABI call (visible in nsys / ncu timelines; a no-op without a tool attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// First block (a multiple of 32) from which k_chain_probe probes a tile in two waves: the tile
// expected to hold a large batch's first misses (the previous batch's mean match length), so the
// probes past a miss shrink without adding rounds to the all-found tiles before it.  Performance
// only: every choice gives the same results.
uint32_t probe_split_from(const skv_ctx* c, uint32_t N) {
  static const char* force = std::getenv("SKV_PROBE_SPLIT");  // diagnostic / tests: a fixed split block
  if (force) return static_cast<uint32_t>(std::strtoul(force, nullptr, 10));
  if (N < 16384 || c->probe_est < 0) return UINT32_MAX;
  if (c->probe_est < 24) return 0;
  if (c->probe_est < 64) return 32;
  return UINT32_MAX;
}

// an event record inside a captured phase is an external event node (its timestamps stay
// readable after the graph ran)
void rec_ev(skv_ctx* c, cudaEvent_t e, cudaStream_t s) {
  CK(c->capturing ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal) : cudaEventRecord(e, s));
}

// the device step state of phase `slot` (0 admit, 1 commit, 2 epoch) from the host mirrors
void put_state(skv_ctx* c, int slot, uint32_t batch, uint64_t epoch, bool armed = false) {
  uint32_t* h = c->hstate + 8 * slot;
  h[0] = batch;
  h[1] = c->wstart;
  h[2] = static_cast<uint32_t>(c->cur);
  h[3] = static_cast<uint32_t>(epoch);
  h[4] = static_cast<uint32_t>(epoch);
  h[5] = static_cast<uint32_t>(epoch >> 32);
  h[6] = armed ? 1u : 0u;  // a speculative epoch pass (skv_step)
  CK(cudaMemcpyAsync(c->dstate, h, 7 * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
}

// Replay `issue` (the phase's launches) from its graph, capturing it first when the key (the
// buffers and shapes the launches bake in) changed.
template <typename F>
void run_graph(skv_ctx* c, skv_ctx::GraphCache& g, const std::vector<uintptr_t>& key, F&& issue) {
  constexpr size_t kKeep = 4;  // e.g. alternating batch shapes / buffers replay without re-capture
  cudaStream_t s = c->stream;
  auto hit = std::find_if(g.items.begin(), g.items.end(), [&](const auto& it) { return it.key == key; });
  if (hit == g.items.end()) {
    cudaGraph_t graph = nullptr;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    c->capturing = true;
    try {
      issue();
    } catch (...) {
      c->capturing = false;
      cudaStreamEndCapture(s, &graph);
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      throw;
    }
    c->capturing = false;
    CK(cudaStreamEndCapture(s, &graph));
    cudaGraphExec_t exec = nullptr;
    const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    CK(e);
    if (g.items.size() == kKeep) {
      cudaGraphExecDestroy(g.items.back().exec);
      g.items.pop_back();
    }
    g.items.insert(g.items.begin(), skv_ctx::GraphCache::Item{exec, key});
    hit = g.items.begin();
  } else if (hit != g.items.begin()) {
    std::rotate(g.items.begin(), hit, hit + 1);
    hit = g.items.begin();
  }
  CK(cudaGraphLaunch(hit->exec, s));
}

void check_usable(const skv_ctx* c) {
  if (!c->poisoned.empty()) throw StateError("context unusable after an earlier failure: " + c->poisoned);
}

// A rule set's device automata (consecutive groups, none straddling a 32-rule mask word) and,
// up to 32 enabled rules, the whole set's automaton (skv_rules_dfa).  Larger libraries keep
// bit j = j-th enabled rule across skv_rules_mask_words() u32 words per window.
void compile_set(skv_rules& r) {
  r.enabled.clear();
  for (size_t i = 0; i < r.spec.rules.size(); ++i)
    if (r.spec.rules[i].enabled) r.enabled.push_back(static_cast<uint32_t>(i));
  if (r.enabled.size() > 32ull * SKV_MAX_MASK_WORDS)
    throw skv::CompileError("rule set has " + std::to_string(r.enabled.size()) + " enabled rules (device maximum " +
                            std::to_string(32 * SKV_MAX_MASK_WORDS) + ")");
  r.groups = skv::compile_rule_groups(r.spec.rules, fits_device);
  r.whole = r.enabled.size() <= 32;
  r.dfa = r.whole ? skv::compile_rules(r.spec.rules) : skv::DfaTables{};
}

}  // namespace

extern "C" {

// ------------------------------------------------------------------ rules
int skv_rules_default(skv_rules** out) {
  if (!out) return SKV_ERR_ARG;
  return guard(nullptr, [&] {
    auto r = std::make_unique<skv_rules>();
    r->spec.version = 1;  // RuleEngine() default snapshot version (detection.hpp:210)
    r->spec.rules = skv::default_pattern_rules();
    compile_set(*r);
    *out = r.release();
    return SKV_OK;
  });
}

int skv_rules_from_json(const char* json, size_t len, skv_rules** out, char* err, size_t errcap) {
  if (!json || !out) return SKV_ERR_ARG;
  skv_ctx scratch;  // carries the error message
  int rc = guard(&scratch, [&] {
    auto r = std::make_unique<skv_rules>();
    r->spec = skv::parse_rules_json(std::string(json, len));
    compile_set(*r);
    *out = r.release();
    return SKV_OK;
  });
  if (rc != SKV_OK && err && errcap) {
    size_t n = std::min(errcap - 1, scratch.err.size());
    std::memcpy(err, scratch.err.data(), n);
    err[n] = 0;
  }
  return rc;
}

void skv_rules_free(skv_rules* r) { delete r; }
uint64_t skv_rules_version(const skv_rules* r) { return r ? r->spec.version : 0; }
uint32_t skv_rules_count(const skv_rules* r) { return r ? static_cast<uint32_t>(r->spec.rules.size()) : 0; }

int skv_rules_info(const skv_rules* r, uint32_t i, const char** rule_id, const char** category, int* kind,
                   int* enabled) {
  if (!r || i >= r->spec.rules.size()) return SKV_ERR_ARG;
  const auto& x = r->spec.rules[i];
  if (rule_id) *rule_id = x.rule_id.c_str();
  if (category) *category = x.category.c_str();
  if (kind) *kind = x.blacklist ? 1 : 0;
  if (enabled) *enabled = x.enabled ? 1 : 0;
  return SKV_OK;
}

size_t skv_rules_warning_count(const skv_rules* r) { return r ? r->spec.warnings.size() : 0; }
const char* skv_rules_warning(const skv_rules* r, size_t i) {
  return (r && i < r->spec.warnings.size()) ? r->spec.warnings[i].c_str() : nullptr;
}
uint32_t skv_rules_group_count(const skv_rules* r) {
  return r ? static_cast<uint32_t>(r->groups.groups.size()) : 0;
}

uint32_t skv_rules_enabled_count(const skv_rules* r) { return r ? static_cast<uint32_t>(r->enabled.size()) : 0; }
uint32_t skv_rules_enabled_rule(const skv_rules* r, uint32_t j) {
  return (r && j < r->enabled.size()) ? r->enabled[j] : UINT32_MAX;
}
uint32_t skv_rules_mask_words(const skv_rules* r) { return r ? mask_words_of(*r) : 0; }

int skv_rules_dfa(const skv_rules* r, skv_dfa_view* v) {
  if (!r || !v) return SKV_ERR_ARG;
  if (!r->whole) return SKV_ERR_COMPILE;  // more than 32 enabled rules: no single automaton
  v->n_states = r->dfa.n_states;
  v->n_classes = r->dfa.n_classes;
  v->start = r->dfa.start;
  v->class_map = r->dfa.class_map;
  v->next = r->dfa.next.data();
  v->acc = r->dfa.acc.data();
  v->nfa_states = r->dfa.nfa_states;
  v->dfa_states_unminimized = r->dfa.dfa_states_unminimized;
  return SKV_OK;
}

// ------------------------------------------------------------------ context
void skv_config_default(skv_config* c) {
  if (!c) return;
  c->device = 0;
  c->block_tokens = 16;
  c->window_tokens = 32;
  c->index_capacity = 1ull << 20;
  c->max_prompts = 1ull << 16;
  c->max_tokens = 1ull << 24;
  c->max_window_entries = 1ull << 16;
  c->entropy_jump = 0.3;  // MonitorConfig defaults (monitor.hpp:12-15)
  c->u_pre_max = 1;
  c->max_users = 1ull << 20;
}

int skv_create(const skv_config* cfg, skv_ctx** out) {
  if (!cfg || !out) return SKV_ERR_ARG;
  auto c = std::make_unique<skv_ctx>();
  int rc = guard(c.get(), [&] {
    c->cfg = *cfg;
    const uint32_t B = cfg->block_tokens;
    if (B < 1 || B > 4096) throw skv::ConfigError("block_tokens must be in [1, 4096]");
    if (cfg->window_tokens > 4096) throw skv::ConfigError("window_tokens must be <= 4096");
    if (cfg->max_prompts == 0 || cfg->max_prompts > skv::kMaxBatchPrompts)
      throw skv::ConfigError("max_prompts must be in [1, 2^24]");
    if (cfg->max_users == 0 || cfg->max_users >= (1ull << 30)) throw skv::ConfigError("bad max_users");
    if (cfg->max_tokens / B >= (1ull << 31)) throw skv::ConfigError("max_tokens / block_tokens must be < 2^31");
    if (cfg->max_window_entries == 0 || cfg->max_window_entries >= (1ull << 31))
      throw skv::ConfigError("bad max_window_entries");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
      throw CudaError("no CUDA device available (this library has no CPU fallback)");
    if (cfg->device < 0 || cfg->device >= ndev) throw skv::ConfigError("device ordinal out of range");
    c->device = cfg->device;
    CK(cudaSetDevice(c->device));
    cudaDeviceProp prop{};
    CK(cudaGetDeviceProperties(&prop, c->device));
    if (prop.major != 10)
      throw CudaError("device " + std::string(prop.name) + " is not sm_100 (built for sm_100a only)");
    c->n_sm = prop.multiProcessorCount;
    {
      // SKV_STREAM_PRIO (diagnostic): 1 = the batch's own work (admit, commit, epoch) ahead of the
      // next batch's prefetch when both have CTAs waiting, 2 = the prefetch ahead
      const char* pe = std::getenv("SKV_STREAM_PRIO");
      const int mode = pe ? std::atoi(pe) : SKV_STREAM_PRIO;
      int prio_lo = 0, prio_hi = 0;
      CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
      CK(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, mode == 1 ? prio_hi : prio_lo));
      CK(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, mode == 2 ? prio_hi : prio_lo));
    }
    CK(cudaStreamCreateWithFlags(&c->rec_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->rec_start, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->rec_done, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->pf_done, cudaEventDisableTiming));
    for (auto& pr : c->pf_ev)
      for (auto& ev : pr) CK(cudaEventCreate(&ev));
    for (auto& ev : c->ev) CK(cudaEventCreate(&ev));
    // index
    uint64_t cap = next_pow2(std::max<uint64_t>(cfg->index_capacity, 1024));
    if (cap > (1ull << 31)) throw skv::ConfigError("index_capacity must be <= 2^31");
    c->cfg.index_capacity = cap;
    c->ix.cap = cap;
    c->ix.mask = cap - 1;
    c->ix.e = dalloc<skv::Entry>(cap, c->owned);
    skv::launch_init_entries(c->ix, c->stream);
    // monitor window
    c->pool_cap = static_cast<uint32_t>(cfg->max_window_entries);
    c->set_hdr = dalloc<skv::SetHdr>(c->pool_cap, c->owned);
    c->set_tab = dalloc<ulonglong2>(static_cast<size_t>(c->pool_cap) * skv::kSetSlots, c->owned);
    // slots are live by their window stamp: a fresh pool must hold none (memory reused from an
    // earlier context would otherwise carry its stamps)
    CK(cudaMemsetAsync(c->set_tab, 0, static_cast<size_t>(c->pool_cap) * skv::kSetSlots * sizeof(ulonglong2), c->stream));
    CK(cudaMemsetAsync(c->set_hdr, 0, static_cast<size_t>(c->pool_cap) * sizeof(skv::SetHdr), c->stream));
    c->replay = dalloc<uint32_t>(c->pool_cap, c->owned);
    c->touched[0] = dalloc<uint32_t>(c->pool_cap, c->owned);
    c->touched[1] = dalloc<uint32_t>(c->pool_cap, c->owned);
    c->counters = dalloc<uint32_t>(16, c->owned);
    c->n_new = dalloc<unsigned long long>(1, c->owned);
    CK(cudaMemsetAsync(c->counters, 0, 16 * sizeof(uint32_t), c->stream));
    c->cands = dalloc<uint32_t>(2ull * c->pool_cap, c->owned);
    c->fired = dalloc<uint32_t>(2ull * c->pool_cap, c->owned);
    c->events = dalloc<skv_event>(2ull * c->pool_cap, c->owned);
    // the epoch reads back its first kEpochEvPre slots with the count (defined contents)
    CK(cudaMemset(c->events, 0, std::min<size_t>(kEpochEvPre, 2ull * c->pool_cap) * sizeof(skv_event)));
    // batch buffers
    c->max_prompts = cfg->max_prompts;
    c->max_tokens = cfg->max_tokens;
    c->max_blocks = cfg->max_tokens / B;
    const uint64_t N = c->max_prompts, NB = std::max<uint64_t>(c->max_blocks, 1);
    c->d_tokens = dalloc<uint32_t>(c->max_tokens + 4, c->owned);
    c->d_off = dalloc<uint64_t>(N + 1, c->owned);
    c->d_users = dalloc<uint64_t>(N, c->owned);
    c->d_owners = dalloc<uint8_t>(N, c->owned);
    c->counts = dalloc<uint32_t>(N + 1, c->owned);
    c->blk_off = dalloc<uint32_t>(N + 1, c->owned);
    c->first_sens = dalloc<uint32_t>(N, c->owned);
    c->matched = dalloc<uint32_t>(N + 1, c->owned);
    c->exist = dalloc<uint32_t>(N, c->owned);
    c->tier = dalloc<uint8_t>(N, c->owned);
    c->bh = dalloc<uint64_t>(NB, c->owned);
    c->bd = dalloc<uint64_t>(NB, c->owned);
    c->bmask = dalloc<uint32_t>(NB, c->owned);
    c->alt_counts = dalloc<uint32_t>(N + 1, c->owned);
    c->alt_blk_off = dalloc<uint32_t>(N + 1, c->owned);
    c->alt_first_sens = dalloc<uint32_t>(N, c->owned);
    c->alt_bd = dalloc<uint64_t>(NB, c->owned);
    c->alt_bh = dalloc<uint64_t>(NB, c->owned);
    c->alt_blabel = dalloc<uint8_t>(NB, c->owned);
    c->alt_bslot = dalloc<uint32_t>(NB, c->owned);
    c->alt_bmask = dalloc<uint32_t>(NB, c->owned);
    c->blabel = dalloc<uint8_t>(NB, c->owned);
    c->bprompt = dalloc<uint32_t>(NB, c->owned);
    c->late = dalloc<uint32_t>(2 * NB, c->owned);
    c->bdecision = dalloc<uint8_t>(NB, c->owned);
    c->bslot = dalloc<uint32_t>(NB, c->owned);
    c->bmeta = dalloc<uint8_t>(NB, c->owned);
    c->plen = dalloc<uint32_t>(N, c->owned);
    c->alt_plen = dalloc<uint32_t>(N, c->owned);
    c->d_ttft = dalloc<double>(N, c->owned);
    c->d_intra = dalloc<uint32_t>(N, c->owned);
    c->d_inter = dalloc<uint32_t>(N, c->owned);
    c->d_reqid = dalloc<uint64_t>(N, c->owned);
    c->keys_a = dalloc<unsigned long long>(NB, c->owned);
    c->keys_b = dalloc<unsigned long long>(NB, c->owned);
    c->fix_list = dalloc<uint32_t>(4 * NB, c->owned);
    c->uidx = dalloc<uint32_t>(N, c->owned);
    {  // user table: 2x slots, keys = kNoUser, idx = 0, index 0 reserved for UserId ~0
      uint32_t slots = 1;
      while (slots < 2 * cfg->max_users) slots <<= 1;
      c->users_tab.keys = dalloc<unsigned long long>(slots, c->owned);
      c->users_tab.idx = dalloc<uint32_t>(slots, c->owned);
      c->users_tab.rev = dalloc<uint64_t>(cfg->max_users + 1, c->owned);
      c->users_tab.count = dalloc<uint32_t>(1, c->owned);
      c->users_tab.mask = slots - 1;
      c->users_tab.cap = static_cast<uint32_t>(cfg->max_users + 1);
      CK(cudaMemsetAsync(c->users_tab.keys, 0xff, slots * 8ull, c->stream));
      CK(cudaMemsetAsync(c->users_tab.idx, 0, slots * 4ull, c->stream));
      CK(cudaMemsetAsync(c->users_tab.rev, 0xff, 8, c->stream));
      CK(cudaMemsetAsync(c->users_tab.count, 0, 4, c->stream));
    }
    size_t tb = std::max(skv::scan_temp_bytes(static_cast<uint32_t>(std::max(N + 1, NB))),
                         skv::sort_keys_temp_bytes(static_cast<uint32_t>(NB), 32 + log2u(cap)));
    c->temp_bytes = tb;
    c->side_temp_bytes = skv::scan_temp_bytes(static_cast<uint32_t>(N + 1));
    c->side_temp = dalloc<uint8_t>(c->side_temp_bytes, c->owned);
    c->temp = dalloc<uint8_t>(tb, c->owned);
    CK(cudaMallocHost(&c->host_small, 64 * sizeof(uint32_t)));
    CK(cudaMallocHost(&c->host_events, kEpochEvPre * sizeof(skv_event)));
    CK(cudaMallocHost(&c->hstate, 24 * sizeof(uint32_t)));
    c->dstate = dalloc<uint32_t>(8, c->owned);
    CK(cudaMemsetAsync(c->dstate, 0, 8 * sizeof(uint32_t), c->stream));
    c->graphs = !(std::getenv("SKV_GRAPHS") && std::atoi(std::getenv("SKV_GRAPHS")) == 0);
    c->rec_grid = skv::record_grid(c->device);
    // default rules
    skv_rules* r = nullptr;
    int rr = skv_rules_default(&r);
    if (rr != SKV_OK) throw skv::CompileError("default rules failed to compile");
    std::unique_ptr<skv_rules> hold(r);
    upload_rules(c.get(), *r);
    sync_check(c->stream);
    return SKV_OK;
  });
  if (rc != SKV_OK) {
    // the ctx is destroyed: keep the message for skv_last_error(NULL)
    g_create_err = c->err;
    for (void* p : c->owned) cudaFree(p);
    c->owned.clear();
    *out = nullptr;
    return rc;
  }
  *out = c.release();
  return SKV_OK;
}

int find_staged(skv_ctx* c, const skv_batch* b);
void unprefetch_slot(skv_ctx* c);

int skv_stage(skv_ctx* c, const skv_batch* b) {
  NvtxRange nvtx_range("skv_stage");
  if (!c || !b) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    if (b->on_device) throw ArgError("skv_stage: host batches only");
    const uint32_t N = b->n_prompts;
    if (N > c->max_prompts) throw ArgError("n_prompts exceeds max_prompts");
    if (b->n_tokens > c->max_tokens) throw ArgError("n_tokens exceeds max_tokens");
    if (N == 0 || (!b->tokens && !b->token_bytes) || !b->offsets || !b->users) return SKV_OK;
    if (find_staged(c, b) >= 0) return SKV_OK;
    int si = -1;
    for (int i = 0; i < skv_ctx::kHostSlots && si < 0; ++i)
      if (c->hslot[i].state == skv_ctx::kSlotFree) si = i;
    if (si < 0) return SKV_OK;  // every slot busy: the prefetch / admit copies it inline
    auto& hs = c->hslot[si];
    if (!c->copy) CK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
    if (!hs.tok) {
      hs.tok = dalloc<uint32_t>(c->max_tokens + 4, c->owned);
      hs.tok8 = dalloc<uint8_t>(c->max_tokens + 16, c->owned);
      hs.off = dalloc<uint64_t>(c->max_prompts + 1, c->owned);
      hs.users = dalloc<uint64_t>(c->max_prompts, c->owned);
      hs.owners = dalloc<uint8_t>(c->max_prompts, c->owned);
      CK(cudaEventCreateWithFlags(&hs.ready, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&hs.free_ev, cudaEventDisableTiming));
    }
    cudaStream_t cs = c->copy;
    CK(cudaStreamWaitEvent(cs, hs.free_ev, 0));  // the slot's last reader (a previous batch's commit)
    if (b->token_bytes)
      CK(cudaMemcpyAsync(hs.tok8, b->token_bytes, b->n_tokens, cudaMemcpyHostToDevice, cs));
    else
      CK(cudaMemcpyAsync(hs.tok, b->tokens, b->n_tokens * 4, cudaMemcpyHostToDevice, cs));
    CK(cudaMemcpyAsync(hs.off, b->offsets, (N + 1) * 8ull, cudaMemcpyHostToDevice, cs));
    CK(cudaMemcpyAsync(hs.users, b->users, N * 8ull, cudaMemcpyHostToDevice, cs));
    if (b->owners) CK(cudaMemcpyAsync(hs.owners, b->owners, N, cudaMemcpyHostToDevice, cs));
    CK(cudaEventRecord(hs.ready, cs));
    hs.state = skv_ctx::kSlotStaged;
    hs.id_tok = b->token_bytes ? static_cast<const void*>(b->token_bytes) : b->tokens;
    hs.id_off = b->offsets;
    hs.id_users = b->users;
    hs.id_owners = b->owners;
    hs.n = N;
    hs.ntok = b->n_tokens;
    hs.bytes = b->token_bytes != nullptr;
    return SKV_OK;
  });
}

int skv_destroy(skv_ctx* c) {
  if (!c) return SKV_ERR_ARG;
  if (c->copy) cudaStreamSynchronize(c->copy);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->side) cudaStreamSynchronize(c->side);
  if (c->rec_stream) cudaStreamSynchronize(c->rec_stream);
  for (void* p : c->owned) cudaFree(p);
  for (auto& g : c->groups) free_group(g);
  for (void* p : {c->rep_in, static_cast<void*>(c->rep_slots), static_cast<void*>(c->rep_uidx)})
    if (p) cudaFree(p);
  if (c->host_small) cudaFreeHost(c->host_small);
  if (c->host_events) cudaFreeHost(c->host_events);
  if (c->hstate) cudaFreeHost(c->hstate);
  for (auto* g : {&c->g_admit, &c->g_commit, &c->g_epoch})
    for (auto& it : g->items)
      if (it.exec) cudaGraphExecDestroy(it.exec);
  for (auto& ev : c->ev)
    if (ev) cudaEventDestroy(ev);
  if (c->side) {
    cudaStreamSynchronize(c->side);
    cudaStreamDestroy(c->side);
  }
  if (c->rec_stream) cudaStreamDestroy(c->rec_stream);
  if (c->rec_start) cudaEventDestroy(c->rec_start);
  if (c->rec_done) cudaEventDestroy(c->rec_done);
  if (c->pf_done) cudaEventDestroy(c->pf_done);
  for (auto& pr : c->pf_ev)
    for (auto ev : pr)
      if (ev) cudaEventDestroy(ev);
  if (c->stream) cudaStreamDestroy(c->stream);
  for (auto& h : c->hslot) {
    if (h.ready) cudaEventDestroy(h.ready);
    if (h.free_ev) cudaEventDestroy(h.free_ev);
  }
  if (c->copy) cudaStreamDestroy(c->copy);
  delete c;
  return SKV_OK;
}

const char* skv_last_error(const skv_ctx* c) { return c ? c->err.c_str() : g_create_err.c_str(); }

int skv_set_rules(skv_ctx* c, const skv_rules* r) {
  if (!c || !r) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    if (c->pf_valid) CK(cudaStreamSynchronize(c->side));
    if (c->pf_valid) unprefetch_slot(c);
    c->pf_valid = false;  // a staged scan used the previous rule snapshot
    upload_rules(c, *r);
    return SKV_OK;
  });
}

void* skv_stream(skv_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

// ------------------------------------------------------------------ monitor records
// AccessStats::record of the last admitted batch (A.6): the per-access part ran inside
// k_commit (or k_record); this applies the distinct-user counts and replays, in prompt
// order, the rare entries whose tracked set crossed 64 users in the batch.
// Enqueue the distinct-count pass; the caller reads counters[8] (replay count) and
// counters[5] (errors) back with its own synchronisation and calls replay_record.
void finish_record(skv_ctx* c, cudaStream_t s) {
  skv::launch_record_finish(c->ix, c->rec_mon, c->replay, c->counters + 8, static_cast<int>(c->rec_grid), s);
}

uint32_t replay_record(skv_ctx* c, cudaStream_t s, uint32_t n_replay, uint32_t err) {
  const skv::MonCtx& mon = c->rec_mon;
  uint32_t launched = 1;
  c->rec_pending = false;
  if (err & 1u) throw CapacityError("monitor window user-set pool exhausted (raise max_window_entries)");
  c->times.replayed_entries = n_replay;
  if (n_replay > 0) {
    skv::launch_replay_emit(c->ix, mon, c->bslot, c->blk_off, c->matched, c->rec_n, c->keys_a, c->counters + 9, s);
    CK(cudaMemcpyAsync(c->host_small, c->counters + 9, 4, cudaMemcpyDeviceToHost, s));
    sync_check(s);
    const uint32_t nk = c->host_small[0];
    const int end_bit = 32 + log2u(c->ix.cap);
    skv::launch_sort_keys(c->temp, c->temp_bytes, c->keys_a, c->keys_b, nk, end_bit, s);
    skv::launch_record_replay(c->ix, mon, c->replay, c->counters + 8, c->keys_b, nk, c->rec_users,
                              static_cast<int>(c->rec_grid), s);
    launched += 2 + 2 + (end_bit + 7) / 8;
  }
  return launched;
}

// records of a batch that is not committed (next admit, epoch or export first)
void flush_record(skv_ctx* c) {
  if (!c->rec_pending) return;
  // a replicated layer aggregates the batch's accesses for the cross-rank merge, which follows
  // the batch's commit: an uncommitted batch cannot be merged
  if (c->ix.rep.depth) throw StateError("replicated layer: commit the admitted batch first");
  c->rec_mon.st = nullptr;  // outside a graph: the host's stamps
  c->adm_graph = false;
  cudaStream_t s = c->stream;
  skv::launch_record(c->ix, c->rec_mon, c->bslot, c->blk_off, c->matched, c->rec_users, c->rec_n, s);
  finish_record(c, s);
  CK(cudaMemcpyAsync(c->host_small, c->counters + 8, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(c->host_small + 1, c->counters + 5, 4, cudaMemcpyDeviceToHost, s));
  sync_check(s);
  replay_record(c, s, c->host_small[0], c->host_small[1]);
}

// ------------------------------------------------------------------ admission
void resolve_admit(skv_ctx* c);

// a lazily admitted batch's readbacks must have landed before the host looks at them
void ensure_admit_resolved(skv_ctx* c) {
  if (!c->adm_lazy) return;
  sync_check(c->stream);
  resolve_admit(c);
}

// ------------------------------------------------------------------ host staging ring
int find_staged(skv_ctx* c, const skv_batch* b) {
  const void* tok = b->token_bytes ? static_cast<const void*>(b->token_bytes) : b->tokens;
  for (int i = 0; i < skv_ctx::kHostSlots; ++i) {
    const auto& h = c->hslot[i];
    if (h.state == skv_ctx::kSlotStaged && h.id_tok == tok && h.id_off == b->offsets && h.id_users == b->users &&
        h.id_owners == b->owners && h.n == b->n_prompts && h.ntok == b->n_tokens && h.bytes == (b->token_bytes != nullptr))
      return i;
  }
  return -1;
}

// the pending batch no longer reads its slot once the kernels queued so far have run
void release_slot(skv_ctx* c) {
  if (c->use_slot < 0) return;
  auto& h = c->hslot[c->use_slot];
  CK(cudaEventRecord(h.free_ev, c->stream));
  h.state = skv_ctx::kSlotFree;
  c->use_slot = -1;
}

// a dropped prefetch leaves its staged copy usable
void unprefetch_slot(skv_ctx* c) {
  if (c->pf_slot >= 0 && c->hslot[c->pf_slot].state == skv_ctx::kSlotPrefetched)
    c->hslot[c->pf_slot].state = skv_ctx::kSlotStaged;
  c->pf_slot = -1;
}

int skv_admit(skv_ctx* c, const skv_batch* b, skv_admit_out* out) {
  NvtxRange nvtx_range("skv_admit");
  if (!c || !b) return SKV_ERR_ARG;
  return guard(c, [&] {
    check_usable(c);
    CK(cudaSetDevice(c->device));
    const uint32_t N = b->n_prompts;
    const uint32_t B = c->cfg.block_tokens;
    if (N > c->max_prompts) throw ArgError("n_prompts exceeds max_prompts");
    if (b->n_tokens > c->max_tokens) throw ArgError("n_tokens exceeds max_tokens");
    if (c->rep_sync_due) throw StateError("replicated layer: skv_replica_export / skv_replica_apply of the last batch first");
    ensure_admit_resolved(c);
    flush_record(c);  // the previous batch was admitted but not committed
    release_slot(c);
    c->dropped_by_evict = false;
    if (N == 0) {
      if (out) out->n_blocks = 0, out->matched_total = 0;
      c->pending = true;
      c->p_n = 0;
      c->p_blocks = 0;
      c->last_n = 0;
      return SKV_OK;
    }
    if ((!b->tokens && !b->token_bytes) || !b->offsets || !b->users) throw ArgError("null batch pointer");
    const void* tok_id = b->token_bytes ? static_cast<const void*>(b->token_bytes) : b->tokens;
    cudaStream_t s = c->stream;
    const uint32_t* tokens;
    const uint64_t* off;
    const uint64_t* users;
    const uint8_t* owners;
    uint64_t n_blocks = 0;
    // stages 1+2 (and for host batches the H2D) were staged by skv_prefetch for exactly this batch?
    const bool use_pf = c->pf_valid && c->pf_on_device == (b->on_device != 0) && c->pf_tokens == tok_id &&
                        c->pf_offsets == b->offsets && c->pf_users == b->users && c->pf_owners == b->owners &&
                        c->pf_n == N && c->pf_ntok == b->n_tokens;
    if (c->pf_valid && !use_pf) {  // stale prefetch: drop it
      CK(cudaStreamSynchronize(c->side));
      unprefetch_slot(c);
    }
    c->pf_valid = false;
    c->adm_graph = false;
    // a small device batch without per-block outputs: the admit's launches replay from a graph
    if (c->graphs && b->on_device && !use_pf && !out && !c->evict_on && !c->budget_on && !c->ix.rep.depth) {
      c->pf_slot = -1;
      const bool bytes = b->token_bytes != nullptr;
      const bool unaligned = !bytes && reinterpret_cast<uintptr_t>(b->tokens) % 16 != 0;
      const uint32_t* tokens = (bytes || unaligned) ? c->d_tokens : b->tokens;
      const uint64_t nb_bound = b->n_tokens / B;
      const uint32_t split = probe_split_from(c, N);
      skv::MonCtx mon = monitor_ctx(c);
      mon.st = c->dstate;
      mon.tl[0] = c->touched[0];
      mon.tl[1] = c->touched[1];
      mon.ntb = c->counters + 1;
      const std::vector<uintptr_t> key = {
          reinterpret_cast<uintptr_t>(bytes ? static_cast<const void*>(b->token_bytes) : b->tokens),
          reinterpret_cast<uintptr_t>(b->offsets), reinterpret_cast<uintptr_t>(b->users),
          reinterpret_cast<uintptr_t>(b->owners), N, b->n_tokens, reinterpret_cast<uintptr_t>(c->bd),
          reinterpret_cast<uintptr_t>(c->bh), reinterpret_cast<uintptr_t>(c->bmask),
          reinterpret_cast<uintptr_t>(c->blk_off), reinterpret_cast<uintptr_t>(c->first_sens),
          reinterpret_cast<uintptr_t>(c->bslot), reinterpret_cast<uintptr_t>(c->blabel),
          reinterpret_cast<uintptr_t>(c->counts), reinterpret_cast<uintptr_t>(c->plen), c->rules_gen, c->mask_words,
          static_cast<uintptr_t>(bytes), static_cast<uintptr_t>(unaligned), split};
      put_state(c, 0, mon.batch, c->epoch);
      run_graph(c, c->g_admit, key, [&] {
        rec_ev(c, c->ev[0], s);
        if (bytes)
          skv::launch_widen(b->token_bytes, c->d_tokens, b->n_tokens, s);
        else if (unaligned)
          CK(cudaMemcpyAsync(c->d_tokens, b->tokens, b->n_tokens * 4, cudaMemcpyDeviceToDevice, s));
        skv::launch_block_counts(b->offsets, N, B, c->counts, c->plen, s);
        skv::launch_exclusive_scan(c->temp, c->temp_bytes, c->counts, c->blk_off, N + 1, s);
        CK(cudaMemsetAsync(c->first_sens, 0xff, N * 4ull, s));
        CK(cudaMemsetAsync(c->bdecision, 0, std::max<uint64_t>(nb_bound, 1), s));
        CK(cudaMemsetAsync(c->matched + N, 0, 4, s));
        rec_ev(c, c->ev[1], s);
        stage12(c, s, tokens, b->offsets, N, b->n_tokens, nb_bound, c->blk_off, c->first_sens, c->bd, c->bmask);
        rec_ev(c, c->ev[2], s);
        CK(cudaMemsetAsync(c->counters + 8, 0, 12, s));  // n_replay, n_keys, matched_total
        skv::launch_intern_users(c->users_tab, b->users, N, c->uidx, c->counters + 5, s);
        skv::launch_chain_probe(c->ix, c->bd, c->blk_off, c->first_sens, c->uidx, N, c->bh, c->blabel,
                                c->bdecision, c->bslot, c->matched, c->exist, c->tier, c->bmeta, mon, c->bprompt, 0,
                                split, s);
        rec_ev(c, c->ev[3], s);
        rec_ev(c, c->ev[4], s);
        CK(cudaMemcpyAsync(c->host_small + 8, c->counters, 11 * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(c->host_small + 20, c->blk_off + N, 4, cudaMemcpyDeviceToHost, s));
      });
      c->rec_pending = !c->no_record;
      c->rec_mon = mon;
      c->rec_users = b->users;
      c->rec_n = N;
      c->adm_lazy = true;
      c->adm_nb_dev = true;
      c->adm_out = nullptr;
      c->adm_use_pf = false;
      c->adm_pf_pair = c->pf_pair;
      c->adm_launched = 6;
      c->adm_graph = true;
      c->pending = true;
      c->p_n = N;
      c->p_blocks = nb_bound;  // exact after resolve_admit
      c->p_users = b->users;
      c->p_owners = b->owners;
      c->last_n = N;
      c->admitted_prompts += N;
      return SKV_OK;
    }
    CK(cudaEventRecord(c->ev[0], s));
    // the host batch's H2D already queued by skv_stage (and its stages 1-2 by skv_prefetch)?
    int si = -1;
    if (!b->on_device) {
      if (use_pf)
        si = c->pf_slot;
      else
        si = find_staged(c, b);
    }
    c->pf_slot = -1;
    if (si >= 0) {
      n_blocks = host_block_count(b, B);
      auto& hs = c->hslot[si];
      if (!use_pf) {
        CK(cudaStreamWaitEvent(s, hs.ready, 0));
        if (hs.bytes) skv::launch_widen(hs.tok8, hs.tok, b->n_tokens, s);
      }
      tokens = hs.tok;
      off = hs.off;
      users = hs.users;
      owners = b->owners ? hs.owners : nullptr;
      hs.state = skv_ctx::kSlotInUse;
      c->use_slot = si;
    } else if (!b->on_device) {
      n_blocks = host_block_count(b, B);
      if (use_pf) {
        std::swap(c->d_tokens, c->alt_tokens);
        std::swap(c->d_off, c->alt_off);
        std::swap(c->d_users, c->alt_users);
        std::swap(c->d_owners, c->alt_owners);
      } else {
        if (b->token_bytes) {  // byte tokens: a quarter of the copy, widened on the device
          if (!c->d_tok8) c->d_tok8 = dalloc<uint8_t>(c->max_tokens + 16, c->owned);
          CK(cudaMemcpyAsync(c->d_tok8, b->token_bytes, b->n_tokens, cudaMemcpyHostToDevice, s));
          skv::launch_widen(c->d_tok8, c->d_tokens, b->n_tokens, s);
        } else {
          CK(cudaMemcpyAsync(c->d_tokens, b->tokens, b->n_tokens * 4, cudaMemcpyHostToDevice, s));
        }
        CK(cudaMemcpyAsync(c->d_off, b->offsets, (N + 1) * 8ull, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(c->d_users, b->users, N * 8ull, cudaMemcpyHostToDevice, s));
        if (b->owners) CK(cudaMemcpyAsync(c->d_owners, b->owners, N, cudaMemcpyHostToDevice, s));
      }
      tokens = c->d_tokens;
      off = c->d_off;
      users = c->d_users;
      owners = b->owners ? c->d_owners : nullptr;
    } else if (b->token_bytes) {
      if (!use_pf) skv::launch_widen(b->token_bytes, c->d_tokens, b->n_tokens, s);  // else staged by the prefetch
      tokens = c->d_tokens;
      off = b->offsets;
      users = b->users;
      owners = b->owners;
    } else {
      tokens = b->tokens;
      if (reinterpret_cast<uintptr_t>(tokens) % 16) {
        CK(cudaMemcpyAsync(c->d_tokens, b->tokens, b->n_tokens * 4, cudaMemcpyDeviceToDevice, s));
        tokens = c->d_tokens;
      }
      off = b->offsets;
      users = b->users;
      owners = b->owners;
    }
    if (use_pf) {
      CK(cudaStreamWaitEvent(s, c->pf_done, 0));
      std::swap(c->counts, c->alt_counts);
      std::swap(c->plen, c->alt_plen);
      std::swap(c->blk_off, c->alt_blk_off);
      std::swap(c->first_sens, c->alt_first_sens);
      std::swap(c->bd, c->alt_bd);
      std::swap(c->bmask, c->alt_bmask);
      if (kPrefetchChain) {
        std::swap(c->bh, c->alt_bh);
        std::swap(c->blabel, c->alt_blabel);
        std::swap(c->bslot, c->alt_bslot);
      }
    } else {
      skv::launch_block_counts(off, N, B, c->counts, c->plen, s);
      skv::launch_exclusive_scan(c->temp, c->temp_bytes, c->counts, c->blk_off, N + 1, s);
    }
    // a device batch's block count is read back with the admit's single sync at the end
    // (before it only when the caller wants per-block outputs sized by it); until then
    // n_tokens / B bounds it (<= max_blocks since n_tokens <= max_tokens)
    const bool nb_known = !b->on_device;
    if (b->on_device && out) {
      CK(cudaMemcpyAsync(c->host_small, c->blk_off + N, 4, cudaMemcpyDeviceToHost, s));
      sync_check(s);
      n_blocks = c->host_small[0];
    }
    const uint64_t nb_bound = (b->on_device && !out) ? b->n_tokens / B : n_blocks;
    if (!use_pf) CK(cudaMemsetAsync(c->first_sens, 0xff, N * 4ull, s));
    CK(cudaMemsetAsync(c->bdecision, 0, std::max<uint64_t>(nb_bound, 1), s));
    CK(cudaMemsetAsync(c->matched + N, 0, 4, s));
    CK(cudaEventRecord(c->ev[1], s));
    // stages 1+2: digest + rule-tier window scan (unless staged by skv_prefetch)
    if (!use_pf)
      stage12(c, s, tokens, off, N, b->n_tokens, nb_bound, c->blk_off, c->first_sens, c->bd, c->bmask);
    CK(cudaEventRecord(c->ev[2], s));
    // chained keys + labels, then the index probe (stage 3)
    skv::MonCtx mon = monitor_ctx(c);
    CK(cudaMemsetAsync(c->counters + 8, 0, 12, s));  // n_replay, n_keys, matched_total
    skv::launch_intern_users(c->users_tab, users, N, c->uidx, c->counters + 5, s);
    skv::launch_chain_probe(c->ix, c->bd, c->blk_off, c->first_sens, c->uidx, N, c->bh, c->blabel, c->bdecision,
                            c->bslot, c->matched, c->exist, c->tier, c->bmeta, mon, c->bprompt,
                            use_pf && kPrefetchChain ? 1 : 0, probe_split_from(c, N), s);
    if (c->evict_on)  // match_prefix refreshes the access epoch of every visible matched node
      skv::launch_touch_matched(c->ix, c->bslot, c->blk_off, c->matched, N, static_cast<uint32_t>(c->epoch), s);
    CK(cudaEventRecord(c->ev[3], s));
    // stage 4: the monitor records (AccessStats::record of every matched block, in
    // prompt order) run inside the commit kernel, overlapping the claims' DRAM round
    // trips; a batch that is not committed gets them from flush_record
    c->rec_pending = !c->no_record;
    c->rec_mon = mon;
    c->rec_users = users;
    c->rec_n = N;
    uint32_t launched = 6;  // block counts, scan (2), hash/scan, intern, chain/probe
    CK(cudaEventRecord(c->ev[4], s));
    // outputs (per-prompt ones and the summary need no block count)
    if (out) {
      cudaMemcpyKind k = out->on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
      if (out->block_h) CK(cudaMemcpyAsync(out->block_h, c->bh, n_blocks * 8, k, s));
      if (out->block_d) CK(cudaMemcpyAsync(out->block_d, c->bd, n_blocks * 8, k, s));
      if (out->label) CK(cudaMemcpyAsync(out->label, c->blabel, n_blocks, k, s));
      if (out->rule_mask) CK(cudaMemcpyAsync(out->rule_mask, c->bmask, n_blocks * 4, k, s));
      if (out->decision) CK(cudaMemcpyAsync(out->decision, c->bdecision, n_blocks, k, s));
      if (out->matched_blocks) CK(cudaMemcpyAsync(out->matched_blocks, c->matched, N * 4ull, k, s));
      if (out->lowest_tier) CK(cudaMemcpyAsync(out->lowest_tier, c->tier, N, k, s));
      if (out->block_offsets) CK(cudaMemcpyAsync(out->block_offsets, c->blk_off, (N + 1) * 4ull, k, s));
    }
    // counters (errors, touched entries, matched total) and, for a device batch, the
    // block count.  With outputs requested the admit synchronises here; a device batch
    // admitted without outputs does not (the commit that follows is queued right behind
    // it) and these are read with the commit's synchronisation (resolve_admit)
    CK(cudaMemcpyAsync(c->host_small + 8, c->counters, 11 * 4, cudaMemcpyDeviceToHost, s));
    if (!nb_known && !out) CK(cudaMemcpyAsync(c->host_small + 20, c->blk_off + N, 4, cudaMemcpyDeviceToHost, s));
    c->adm_lazy = (!out && b->on_device) || c->lazy_outputs;
    c->adm_nb_dev = !out && b->on_device;
    c->adm_out = c->adm_lazy ? out : nullptr;
    c->adm_use_pf = use_pf;
    c->adm_pf_pair = c->pf_pair;
    c->adm_launched = launched;
    c->pending = true;
    c->p_n = N;
    c->p_blocks = nb_known ? n_blocks : nb_bound;  // exact after resolve_admit
    c->p_users = users;
    c->p_owners = owners;
    c->last_n = N;
    c->admitted_prompts += N;
    if (c->adm_lazy) return SKV_OK;
    sync_check(s);
    resolve_admit(c);
    if (!nb_known) n_blocks = c->p_blocks;
    if (out) {
      out->n_blocks = n_blocks;
      out->matched_total = c->times.matched_total;
    }
    return SKV_OK;
  });
}

// Host-side bookkeeping of the last admit once its readbacks have landed.
void resolve_admit(skv_ctx* c) {
  const uint32_t M = c->host_small[8 + 10];
  if (c->adm_lazy && c->adm_nb_dev) c->p_blocks = c->host_small[20];
  c->adm_lazy = false;
  if (c->adm_out) {  // a lazily admitted batch's output summary (skv_step)
    c->adm_out->n_blocks = c->p_blocks;
    c->adm_out->matched_total = M;
    c->adm_out = nullptr;
  }
  if (c->host_small[8 + 5] & 8u) throw CapacityError("user table exhausted (raise max_users)");
  const bool use_pf = c->adm_use_pf;
  const uint32_t launched = c->adm_launched;
  {
    c->times.hash_scan_ms =
        use_pf ? elapsed(c->pf_ev[c->adm_pf_pair][0], c->pf_ev[c->adm_pf_pair][1]) : elapsed(c->ev[1], c->ev[2]);
    c->times.prefetched = use_pf ? 1 : 0;
    c->times.chain_probe_ms = elapsed(c->ev[2], c->ev[3]);
    c->times.record_ms = elapsed(c->ev[3], c->ev[4]);
    c->times.admit_total_ms = elapsed(c->ev[0], c->ev[4]);
    c->times.matched_total = M;
    c->times.accesses = M;
    if (c->last_n) c->probe_est = static_cast<double>(M) / c->last_n;
    c->times.replayed_entries = 0;
    c->times.touched_entries = c->host_small[8 + 1 + c->cur];
    c->times.kernels_launched = launched;
  }
}

// ------------------------------------------------------------------ serving observables
void skv_cost_model_default(skv_cost_model* m) {
  if (!m) return;
  *m = skv_cost_model{};
  m->t_base_ms = 10.0;  // CostModel defaults (serving_sim.hpp:29-33)
  m->c_prefill_ms = 1.0;
  m->tier_penalty_ms[0] = 0.0;
  m->tier_penalty_ms[1] = 0.2;
  m->tier_penalty_ms[2] = 0.5;
  m->noise_sigma_ms = 0.0;
  m->seed = 0;
}

int skv_set_cost_model(skv_ctx* c, const skv_cost_model* m) {
  if (!c || !m) return SKV_ERR_ARG;
  return guard(c, [&] {
    // CostModel::validate (serving_sim.hpp:35-42)
    if (m->tier_penalty_ms[1] < 0 || m->tier_penalty_ms[2] < m->tier_penalty_ms[1])
      throw skv::ConfigError("cost: tier penalties must satisfy 0 <= DRAM <= SSD");
    if (m->c_prefill_ms <= m->tier_penalty_ms[2])
      throw skv::ConfigError("cost: c_prefill must exceed the SSD reload penalty");
    if (m->noise_sigma_ms < 0) throw skv::ConfigError("cost: noise_sigma must be non-negative");
    c->cost.t_base = m->t_base_ms;
    c->cost.c_prefill = m->c_prefill_ms;
    for (int t = 0; t < 3; ++t) c->cost.penalty[t] = m->tier_penalty_ms[t];
    c->cost.sigma = m->noise_sigma_ms;
    c->cost.seed = m->seed;
    return SKV_OK;
  });
}

int skv_admit_ttft(skv_ctx* c, const uint64_t* request_ids, double* ttft_ms, uint32_t* intra_tokens,
                   uint32_t* inter_tokens, int on_device) {
  if (!c) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    ensure_admit_resolved(c);
    const uint32_t N = c->last_n;
    if (N == 0) return SKV_OK;
    cudaStream_t s = c->stream;
    const cudaMemcpyKind in = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    const cudaMemcpyKind outk = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    const uint64_t* rid = nullptr;
    if (request_ids) {
      CK(cudaMemcpyAsync(c->d_reqid, request_ids, N * 8ull, in, s));
      rid = c->d_reqid;
    }
    skv::launch_ttft(c->blk_off, c->matched, c->plen, c->bmeta, rid, c->admitted_prompts - N, N,
                     c->cfg.block_tokens, c->cost, c->d_ttft, c->d_intra, c->d_inter, s);
    if (ttft_ms) CK(cudaMemcpyAsync(ttft_ms, c->d_ttft, N * 8ull, outk, s));
    if (intra_tokens) CK(cudaMemcpyAsync(intra_tokens, c->d_intra, N * 4ull, outk, s));
    if (inter_tokens) CK(cudaMemcpyAsync(inter_tokens, c->d_inter, N * 4ull, outk, s));
    sync_check(s);
    return SKV_OK;
  });
}

uint32_t skv_mask_words(const skv_ctx* c) { return c ? c->mask_words : 0; }

int skv_access_entropy(skv_ctx* c, uint64_t* h, uint64_t* d, uint64_t* accesses, uint64_t* users, double* bits,
                       size_t cap, size_t* n_entries) {
  if (!c || (cap && (!h || !d || !accesses || !users || !bits))) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    ensure_admit_resolved(c);
    const uint64_t M = c->times.matched_total;
    if (!c->last_n || M == 0) {
      if (n_entries) *n_entries = 0;
      return SKV_OK;
    }
    if (M > 0xffffffffull) throw ArgError("access entropy: batch too large");
    std::vector<void*> tmp;
    const uint32_t w = static_cast<uint32_t>(std::min<size_t>(cap, M));
    uint64_t* dh = dalloc<uint64_t>(std::max<uint32_t>(w, 1), tmp);
    uint64_t* dd = dalloc<uint64_t>(std::max<uint32_t>(w, 1), tmp);
    uint64_t* da = dalloc<uint64_t>(std::max<uint32_t>(w, 1), tmp);
    uint64_t* du = dalloc<uint64_t>(std::max<uint32_t>(w, 1), tmp);
    double* db = dalloc<double>(std::max<uint32_t>(w, 1), tmp);
    uint32_t total = 0, wr = 0;
    try {
      wr = skv::launch_access_entropy(c->ix, c->blk_off, c->matched, c->bslot, c->uidx, c->last_n,
                                      static_cast<uint32_t>(M), dh, dd, da, du, db, w, &total, c->stream);
      if (wr) {
        CK(cudaMemcpy(h, dh, wr * 8ull, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(d, dd, wr * 8ull, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(accesses, da, wr * 8ull, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(users, du, wr * 8ull, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(bits, db, wr * 8ull, cudaMemcpyDeviceToHost));
      }
    } catch (const std::runtime_error& e) {
      for (void* p : tmp) cudaFree(p);
      throw CudaError(e.what());
    }
    for (void* p : tmp) cudaFree(p);
    if (n_entries) *n_entries = total;
    return SKV_OK;
  });
}

int skv_set_graphs(skv_ctx* c, int on) {
  if (!c) return SKV_ERR_ARG;
  c->graphs = on != 0;
  return SKV_OK;
}

int skv_last_rule_masks(skv_ctx* c, uint32_t* out, int on_device) {
  if (!c || !out) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    ensure_admit_resolved(c);
    const uint64_t nb = c->last_n ? c->p_blocks : 0, NB = std::max<uint64_t>(c->max_blocks, 1);
    const cudaMemcpyKind k = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (nb)
      CK(cudaMemcpy2DAsync(out, nb * 4, c->bmask, NB * 4, nb * 4, c->mask_words, k, c->stream));
    sync_check(c->stream);
    return SKV_OK;
  });
}

int skv_prefetch(skv_ctx* c, const skv_batch* b) {
  NvtxRange nvtx_range("skv_prefetch");
  if (!c || !b) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    if (c->pf_valid) {
      CK(cudaStreamSynchronize(c->side));
      unprefetch_slot(c);
    }
    c->pf_valid = false;
    const uint32_t N = b->n_prompts;
    // anything the pipeline cannot stage is admitted inline by skv_admit (which also
    // reports its argument errors)
    if (N == 0 || N > c->max_prompts || b->n_tokens > c->max_tokens || (!b->tokens && !b->token_bytes) ||
        !b->offsets || !b->users)
      return SKV_OK;
    cudaStream_t st = c->side;
    const uint32_t* tokens = b->tokens;
    const uint64_t* off = b->offsets;
    uint64_t nb_hint = 0;
    const int si = b->on_device ? -1 : find_staged(c, b);
    if (si >= 0) {  // copied by skv_stage: stages 1-2 wait for the copy on the device
      try {
        nb_hint = host_block_count(b, c->cfg.block_tokens);
      } catch (const ArgError&) {
        return SKV_OK;
      }
      auto& hs = c->hslot[si];
      CK(cudaStreamWaitEvent(st, hs.ready, 0));
      if (hs.bytes) skv::launch_widen(hs.tok8, hs.tok, b->n_tokens, st);
      tokens = hs.tok;
      off = hs.off;
      hs.state = skv_ctx::kSlotPrefetched;
      c->pf_slot = si;
    } else if (!b->on_device) {
      // host batch: H2D into the alternate staging set on the side stream
      try {
        nb_hint = host_block_count(b, c->cfg.block_tokens);
      } catch (const ArgError&) {
        return SKV_OK;
      }
      if (!c->alt_tokens) {  // allocated on first use (max_tokens x 4 B)
        c->alt_tokens = dalloc<uint32_t>(c->max_tokens + 4, c->owned);
        c->alt_off = dalloc<uint64_t>(c->max_prompts + 1, c->owned);
        c->alt_users = dalloc<uint64_t>(c->max_prompts, c->owned);
        c->alt_owners = dalloc<uint8_t>(c->max_prompts, c->owned);
      }
      if (b->token_bytes) {
        if (!c->alt_tok8) c->alt_tok8 = dalloc<uint8_t>(c->max_tokens + 16, c->owned);
        CK(cudaMemcpyAsync(c->alt_tok8, b->token_bytes, b->n_tokens, cudaMemcpyHostToDevice, st));
        skv::launch_widen(c->alt_tok8, c->alt_tokens, b->n_tokens, st);
      } else {
        CK(cudaMemcpyAsync(c->alt_tokens, b->tokens, b->n_tokens * 4, cudaMemcpyHostToDevice, st));
      }
      CK(cudaMemcpyAsync(c->alt_off, b->offsets, (N + 1) * 8ull, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(c->alt_users, b->users, N * 8ull, cudaMemcpyHostToDevice, st));
      if (b->owners) CK(cudaMemcpyAsync(c->alt_owners, b->owners, N, cudaMemcpyHostToDevice, st));
      tokens = c->alt_tokens;
      off = c->alt_off;
    } else if (b->token_bytes) {  // device byte tokens: widened into the staging set
      if (!c->alt_tokens) {
        c->alt_tokens = dalloc<uint32_t>(c->max_tokens + 4, c->owned);
        c->alt_off = dalloc<uint64_t>(c->max_prompts + 1, c->owned);
        c->alt_users = dalloc<uint64_t>(c->max_prompts, c->owned);
        c->alt_owners = dalloc<uint8_t>(c->max_prompts, c->owned);
      }
      skv::launch_widen(b->token_bytes, c->alt_tokens, b->n_tokens, st);
      tokens = c->alt_tokens;
    } else if (reinterpret_cast<uintptr_t>(b->tokens) % 16) {
      return SKV_OK;
    }
    c->pf_pair ^= 1;
    CK(cudaEventRecord(c->pf_ev[c->pf_pair][0], st));
    skv::launch_block_counts(off, N, c->cfg.block_tokens, c->alt_counts, c->alt_plen, st);
    skv::launch_exclusive_scan(c->side_temp, c->side_temp_bytes, c->alt_counts, c->alt_blk_off, N + 1, st);
    CK(cudaMemsetAsync(c->alt_first_sens, 0xff, N * 4ull, st));
    stage12(c, st, tokens, off, N, b->n_tokens, nb_hint, c->alt_blk_off, c->alt_first_sens, c->alt_bd,
            c->alt_bmask, true);
    // the serial chained-key FNV too, overlapping the current batch's commit; its probe is
    // then lookups only
    if (kPrefetchChain)
      skv::launch_chain(c->alt_bd, c->alt_blk_off, c->alt_first_sens, N, c->alt_bh, c->alt_blabel, c->alt_bslot, st);
    CK(cudaEventRecord(c->pf_done, st));
    CK(cudaEventRecord(c->pf_ev[c->pf_pair][1], st));
    CK(cudaGetLastError());
    c->pf_valid = true;
    c->pf_on_device = b->on_device != 0;
    c->pf_tokens = b->token_bytes ? static_cast<const void*>(b->token_bytes) : b->tokens;
    c->pf_offsets = b->offsets;
    c->pf_users = b->users;
    c->pf_owners = b->owners;
    c->pf_n = N;
    c->pf_ntok = b->n_tokens;
    return SKV_OK;
  });
}

// SMs the persistent commit grid is sized for (SKV_COMMIT_SMS, diagnostic: leave SMs to a
// prefetch running beside it)
int commit_sms(const skv_ctx* c) {
  static const int env = std::getenv("SKV_COMMIT_SMS") ? std::atoi(std::getenv("SKV_COMMIT_SMS")) : 0;
  return env > 0 ? std::min(env, c->n_sm) : c->n_sm;
}

// ------------------------------------------------------------------ A.9 budgeted commit
// Commit of prompts [lo, end) of the pending batch (its monitor records already applied):
// claims + fix-ups, exact node ids, insert-walk epochs.  Returns the entries created.
uint64_t commit_range(skv_ctx* c, uint32_t lo, uint32_t end) {
  if (end <= lo) return 0;
  cudaStream_t s = c->stream;
  const uint32_t n = end - lo;
  const uint32_t ep32 = static_cast<uint32_t>(c->epoch);
  CK(cudaMemsetAsync(c->n_new, 0, 8, s));
  CK(cudaMemsetAsync(c->counters + 7, 0, 4, s));
  CK(cudaMemsetAsync(c->counters + 11, 0, 8, s));
  skv::Index ixc = c->ix;
  skv::launch_node_bases(c->blk_off + lo, c->exist + lo, n, c->ev_counts, c->ev_incl, c->ev_temp, c->ev_temp_bytes, s);
  ixc.em_base = c->ev_incl;
  ixc.em_next = static_cast<uint32_t>(c->node_next);
  ixc.em_epoch = ep32;
  skv::launch_commit(ixc, c->bh, c->bd, c->blk_off + lo, c->exist + lo, c->blabel, c->uidx + lo,
                     c->p_owners ? c->p_owners + lo : nullptr, n, c->bslot, c->n_new, c->fix_list, c->counters + 7,
                     static_cast<uint32_t>(c->max_blocks), c->counters + 5, static_cast<int>(c->rec_grid),
                     c->matched + lo, c->rec_users + lo, nullptr, c->pending_labels ? 1 : 0, c->p_blocks,
                     commit_sms(c), c->bprompt, c->late, c->counters + 11, c->counters + 12, c->rec_mon, s);
  CK(cudaMemcpyAsync(c->host_small, c->n_new, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(c->host_small + 4, c->counters + 5, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(c->host_small + 6, c->counters + 12, 4, cudaMemcpyDeviceToHost, s));
  sync_check(s);
  unsigned long long nn = 0;
  std::memcpy(&nn, c->host_small, 8);
  const uint32_t err = c->host_small[4], revived = c->host_small[6];
  c->entries += nn + revived;
  c->tombstones -= std::min<uint64_t>(c->tombstones, revived);
  if (err) {
    c->node_next += nn + revived;
    const char* why = (err & 2u) ? "index probe sequence exhausted" : "commit fix-up list overflow";
    c->poisoned = why;
    throw CapacityError(why);
  }
  skv::launch_assign_nodes(c->ix, c->bslot, c->blk_off + lo, c->exist + lo, n, c->ev_counts, c->ev_incl, c->node_next,
                           c->ev_temp, c->ev_temp_bytes, s);
  skv::launch_path_epochs(c->ix, c->bslot, c->blk_off + lo, c->exist + lo, n, ep32, s);
  c->node_next += nn + revived;
  return nn + revived;
}

// cap-sized work arrays of one tiered round / tiered evict call (freed by the caller)
skv::TieredWork tiered_work(skv_ctx* c, uint64_t n, std::vector<void*>& tmp) {
  skv::TieredWork w;
  w.cap_each = std::max<uint64_t>(n, 1);
  w.cc = dalloc<uint32_t>(c->ix.cap, tmp);
  w.cc_work = dalloc<uint32_t>(c->ix.cap, tmp);
  w.tier = dalloc<uint8_t>(c->ix.cap, tmp);
  w.keys_a = dalloc<unsigned long long>(3 * w.cap_each, tmp);
  w.keys_b = dalloc<unsigned long long>(3 * w.cap_each, tmp);
  w.hk = dalloc<unsigned long long>(3 * w.cap_each, tmp);
  w.vals_a = dalloc<uint32_t>(3 * w.cap_each, tmp);
  w.vals_b = dalloc<uint32_t>(3 * w.cap_each, tmp);
  w.hv = dalloc<uint32_t>(3 * w.cap_each, tmp);
  w.n3 = dalloc<uint32_t>(3, tmp);
  w.act_cap = 3 * w.cap_each + 16;
  w.act = dalloc<uint32_t>(w.act_cap, tmp);
  w.n_act = dalloc<uint32_t>(1, tmp);
  w.used3 = dalloc<unsigned long long>(4, tmp);
  w.res = dalloc<skv::BudgetSim>(1, tmp);
  w.temp = c->ev_temp;
  w.temp_bytes = c->ev_temp_bytes;
  return w;
}

// host view of a tiered round's result: tier usage, HBM departures, freed entries
struct TieredOutcome {
  skv::BudgetSim r;
  uint64_t used[3], hbm_out, freed;
};

TieredOutcome run_tiered(skv_ctx* c, const uint32_t* vstamp, const uint32_t* needed, uint32_t lo, uint32_t hi,
                         uint64_t need_evict, uint64_t extra) {
  cudaStream_t s = c->stream;
  std::vector<void*> tmp;
  TieredOutcome o{};
  try {
    skv::TieredWork w = tiered_work(c, c->entries + extra + 1, tmp);
    o.r = skv::launch_budget_tiered(c->ix, w, vstamp, needed, lo, hi, need_evict, c->bud_used, c->bud_cap,
                                    static_cast<uint32_t>(c->epoch), c->host_small, s);
    if (o.r.pad) throw CapacityError("tiered budget: action list overflow");
    unsigned long long u[4];
    std::memcpy(u, c->host_small + 8, 32);
    for (int t = 0; t < 3; ++t) o.used[t] = u[t];
    o.hbm_out = u[3];
    // freed entries = live entries that disappeared (count the free actions)
    std::vector<uint32_t> act(o.r.n_victims);
    if (!act.empty()) CK(cudaMemcpyAsync(act.data(), w.act, act.size() * 4, cudaMemcpyDeviceToHost, s));
    sync_check(s);
    for (uint32_t a : act) o.freed += (a >> 30) == 0 ? 1 : 0;
  } catch (...) {
    for (void* p : tmp) cudaFree(p);
    throw;
  }
  for (void* p : tmp) cudaFree(p);
  return o;
}

// The pending batch's commit under a bounded HBM budget (A.9): rounds over prompt ranges, each
// inserting its prompts with the victims their make_room takes (kernels.cu "A.9").
void commit_budgeted(skv_ctx* c) {
  cudaStream_t s = c->stream;
  const uint32_t N = c->p_n;
  const uint32_t E = static_cast<uint32_t>(c->epoch);
  ensure_admit_resolved(c);
  flush_record(c);  // the batch's accesses (prompt order) before its inserts
  c->dropped.clear();
  uint32_t lo = 0;
  while (lo < N) {
    if (lo > 0) skv::launch_reprobe(c->ix, c->bh, c->bd, c->blk_off, lo, N, c->exist, c->bslot, s);
    skv::launch_new_bound(c->blk_off, c->exist, lo, N, c->nb_dev, s);
    CK(cudaMemcpyAsync(c->host_small, c->nb_dev, 8, cudaMemcpyDeviceToHost, s));
    sync_check(s);
    uint64_t bound = 0;
    std::memcpy(&bound, c->host_small, 8);
    uint32_t end = N, next = N, dropped = skv::kNone, nvict = 0;
    if (c->evict_tiered && c->bud_used[0] + bound > c->bud_cap[0]) {  // bounded cascade (kernels.cu)
      CK(cudaMemsetAsync(c->n_mark, 0, 4, s));
      skv::launch_mark_paths(c->bslot, c->blk_off, c->exist, c->matched, lo, N, c->vstamp, c->mark_list, c->n_mark,
                             c->mark_cap, s);
      skv::launch_dry_needed(c->bh, c->bd, c->blk_off, c->exist, lo, N, c->dry_tab, c->dry_minp, c->dry_cap,
                             c->dry_slot, c->needed, s);
      const TieredOutcome o = run_tiered(c, c->vstamp, c->needed, lo, N, 0, c->p_blocks);
      skv::launch_clear_marks(c->vstamp, c->mark_list, c->n_mark, c->mark_cap, s);
      next = o.r.next_lo;
      dropped = o.r.dropped;
      end = dropped != skv::kNone ? dropped : next;
      c->entries -= o.freed;
      c->tombstones += o.freed;
      c->bud_used[0] -= o.hbm_out;
      c->bud_used[1] = o.used[1];
      c->bud_used[2] = o.used[2];
    } else if (c->bud_used[0] + bound > c->bud_cap[0]) {
      CK(cudaMemsetAsync(c->n_mark, 0, 4, s));
      skv::launch_mark_paths(c->bslot, c->blk_off, c->exist, c->matched, lo, N, c->vstamp, c->mark_list, c->n_mark,
                             c->mark_cap, s);
      skv::launch_dry_needed(c->bh, c->bd, c->blk_off, c->exist, lo, N, c->dry_tab, c->dry_minp, c->dry_cap,
                             c->dry_slot, c->needed, s);
      std::vector<void*> tmp;
      try {
        const uint64_t L = std::max<uint64_t>(c->entries, 1);
        auto* keys_a = dalloc<unsigned long long>(L, tmp);
        auto* keys_b = dalloc<unsigned long long>(L, tmp);
        auto* vals_a = dalloc<uint32_t>(L, tmp);
        auto* vals_b = dalloc<uint32_t>(L, tmp);
        auto* victims = dalloc<uint32_t>(L, tmp);
        const uint32_t nv = skv::launch_evict_order(c->ix, c->vstamp, c->ev_eff, keys_a, keys_b, vals_a, vals_b,
                                                    c->ev_n, c->ev_temp, c->ev_temp_bytes, c->host_small, s);
        skv::launch_budget_sim(c->needed, lo, N, c->bud_used[0], c->bud_cap[0], vals_a, nv, c->ev_eff, c->vstamp, E,
                               victims, c->sim, s);
        CK(cudaMemcpyAsync(c->host_small, c->sim, sizeof(skv::BudgetSim), cudaMemcpyDeviceToHost, s));
        sync_check(s);
        skv::BudgetSim r;
        std::memcpy(&r, c->host_small, sizeof(r));
        nvict = r.n_victims;
        next = r.next_lo;
        dropped = r.dropped;
        end = dropped != skv::kNone ? dropped : next;
        skv::launch_clear_marks(c->vstamp, c->mark_list, c->n_mark, c->mark_cap, s);
        skv::launch_evict_mark_list(c->ix, victims, nvict, s);
        sync_check(s);
      } catch (...) {
        for (void* p : tmp) cudaFree(p);
        throw;
      }
      for (void* p : tmp) cudaFree(p);
      c->entries -= nvict;
      c->tombstones += nvict;
      c->bud_used[0] -= nvict;
    }
    const uint64_t made = commit_range(c, lo, end);
    c->bud_used[0] += made;
    if (dropped != skv::kNone) {  // its walk ran before make_room raised (cache_index.hpp:156-176)
      skv::launch_path_epochs(c->ix, c->bslot, c->blk_off + dropped, c->exist + dropped, 1, E, s);
      c->dropped.push_back(dropped);
    }
    if (next <= lo) throw StateError("budgeted commit made no progress");  // cannot happen (kernels.cu A.9)
    lo = next;
  }
}

}  // extern "C"

namespace {

// The non-budgeted commit of the pending batch, enqueued (graph or launches); its readbacks land
// in host_small with the next synchronisation of the stream.
struct CommitRun {
  bool rec;
  uint32_t ep32, launched;
};

CommitRun commit_enqueue(skv_ctx* c) {
  cudaStream_t s = c->stream;
  ++c->batch_id;
  const bool rec = c->rec_pending;  // the batch's monitor records (see skv_admit)
  const uint32_t ep32 = static_cast<uint32_t>(c->epoch);
  // node ids are u32 on the device (the victim order's tie-break); refuse before they wrap
  if (c->evict_on && c->node_next + c->p_blocks >= (1ull << 31))
    throw CapacityError("eviction node-id space exhausted (2^31 nodes created)");
  // a batch admitted through its graph commits through one too (records ride in k_commit)
  const bool graphed = c->graphs && c->adm_graph && !c->evict_on && !c->ix.rep.depth && rec && !kRecordBeside;
  if (!graphed) c->rec_mon.st = nullptr;  // the host's stamps (equal to the device state's)
  uint32_t launched = 4 + (rec && kRecordBeside ? 1 : 0);  // commit, fix-up x2, links
  if (c->evict_on) launched += 2;
  auto issue = [&] {
    rec_ev(c, c->ev[5], s);
    CK(cudaMemsetAsync(c->n_new, 0, 8, s));
    CK(cudaMemsetAsync(c->counters + 7, 0, 4, s));   // intra-batch duplicate fix-up count
    CK(cudaMemsetAsync(c->counters + 11, 0, 8, s));  // late child links, re-inserted tombstones
    if (c->ix.rep.depth) CK(cudaMemsetAsync(c->ix.rep.new_n, 0, 4, s));
    // The records (sector 1 of the matched entries, the window user sets) and the inserts
    // (sector 0 of new entries, first-child links) touch disjoint words, so the record
    // kernel runs on its own stream beside the commit kernels; without it the commit
    // kernel needs fewer registers and keeps more claims in flight.
    if (rec && kRecordBeside) {
      CK(cudaEventRecord(c->rec_start, s));
      CK(cudaStreamWaitEvent(c->rec_stream, c->rec_start, 0));
      skv::launch_record(c->ix, c->rec_mon, c->bslot, c->blk_off, c->matched, c->rec_users, c->rec_n,
                         c->rec_stream);
      CK(cudaEventRecord(c->rec_done, c->rec_stream));
    }
    skv::Index ixc = c->ix;
    if (c->evict_on) {  // speculative node ids: prefix over prompts of the blocks each would create
      skv::launch_node_bases(c->blk_off, c->exist, c->p_n, c->ev_counts, c->ev_incl, c->ev_temp, c->ev_temp_bytes,
                             s);
      ixc.em_base = c->ev_incl;
      ixc.em_next = static_cast<uint32_t>(c->node_next);
      ixc.em_epoch = static_cast<uint32_t>(c->epoch);
    }
    skv::launch_commit(ixc, c->bh, c->bd, c->blk_off, c->exist, c->blabel, c->uidx, c->p_owners, c->p_n, c->bslot,
                       c->n_new, c->fix_list, c->counters + 7, static_cast<uint32_t>(c->max_blocks),
                       c->counters + 5, static_cast<int>(c->rec_grid), c->matched, c->rec_users,
                       rec && !kRecordBeside ? &c->rec_mon : nullptr, c->pending_labels ? 1 : 0, c->p_blocks,
                       commit_sms(c), c->bprompt, c->late, c->counters + 11, c->counters + 12, c->rec_mon, s);
    if (rec && kRecordBeside) CK(cudaStreamWaitEvent(s, c->rec_done, 0));
    if (rec) finish_record(c, s);
    rec_ev(c, c->ev[6], s);
    CK(cudaMemcpyAsync(c->host_small, c->n_new, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(c->host_small + 4, c->counters + 5, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(c->host_small + 5, c->counters + 8, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(c->host_small + 6, c->counters + 12, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(c->host_small + 7, c->counters + 7, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(c->host_small + 44, c->counters + 1, 8, cudaMemcpyDeviceToHost, s));  // both window lists
  };
  if (graphed) {
    const std::vector<uintptr_t> key = {
        c->p_n, c->p_blocks, reinterpret_cast<uintptr_t>(c->rec_users), reinterpret_cast<uintptr_t>(c->p_owners),
        static_cast<uintptr_t>(c->pending_labels), reinterpret_cast<uintptr_t>(c->bh),
        reinterpret_cast<uintptr_t>(c->bd), reinterpret_cast<uintptr_t>(c->blk_off),
        reinterpret_cast<uintptr_t>(c->blabel), reinterpret_cast<uintptr_t>(c->bslot),
        static_cast<uintptr_t>(commit_sms(c)), static_cast<uintptr_t>(c->rec_grid)};
    put_state(c, 1, c->rec_mon.batch, c->epoch);
    run_graph(c, c->g_commit, key, issue);
  } else {
    issue();
  }
  c->adm_graph = false;
  return CommitRun{rec, ep32, launched};
}

// After the synchronisation: errors, the admit's readbacks, the rare ordered replay, counters.
void commit_finish(skv_ctx* c, const CommitRun& run, uint64_t* new_entries) {
  cudaStream_t s = c->stream;
  const bool rec = run.rec;
  const uint32_t ep32 = run.ep32;
  uint32_t launched = run.launched;
  unsigned long long nn = 0;
  std::memcpy(&nn, c->host_small, 8);
  const uint32_t err = c->host_small[4];
  const uint32_t revived = c->host_small[6];
  if (err) {
    // the kernels have run: the host counters follow the device state before anything is
    // raised (skv_export sizes its buffer by them), and the context refuses further batches
    // (its index or monitor state no longer equals the reference's)
    c->entries += nn + revived;
    c->tombstones -= std::min<uint64_t>(c->tombstones, revived);
    c->node_next += nn + revived;
    release_slot(c);
    c->pending = false;
    c->rec_pending = false;
    if (c->adm_lazy && c->adm_nb_dev) c->p_blocks = c->host_small[20];
    c->adm_lazy = false;
    c->adm_out = nullptr;
    const char* why = (err & 8u)   ? "user table exhausted (raise max_users); the batch was not inserted"
                      : (err & 2u) ? "index probe sequence exhausted"
                      : (err & 1u) ? "monitor window user-set pool exhausted (raise max_window_entries)"
                                   : "commit fix-up list overflow";
    if (!(err & 8u)) c->poisoned = why;  // a user-table overflow inserts nothing: still consistent
    else CK(cudaMemsetAsync(c->counters + 5, 0, 4, s));  // ... and the next batch may go ahead
    throw CapacityError(why);
  }
  if (c->adm_lazy) resolve_admit(c);  // the admit's readbacks landed with it
  c->touched_est = c->host_small[44 + c->cur];
  if (rec) launched += replay_record(c, s, c->host_small[5], err);
  if (c->evict_on) {
    // the insert walk refreshes every pre-existing block's access epoch; node ids are exact
    // already unless the batch had duplicate claims
    skv::launch_path_epochs(c->ix, c->bslot, c->blk_off, c->exist, c->p_n, ep32, s);
    launched += 1;
    if (c->host_small[7] || !skv::node_ids_speculative()) {
      skv::launch_assign_nodes(c->ix, c->bslot, c->blk_off, c->exist, c->p_n, c->ev_counts, c->ev_incl,
                               c->node_next, c->ev_temp, c->ev_temp_bytes, s);
      launched += 3;
    }
    c->node_next += nn + revived;
  }
  c->entries += nn + revived;
  c->tombstones -= std::min<uint64_t>(c->tombstones, revived);
  nn += revived;
  c->bud_used[0] += nn;
  c->times.commit_ms = elapsed(c->ev[5], c->ev[6]);
  c->times.kernels_launched += launched;
  c->times.new_blocks = nn;
  release_slot(c);
  c->pending = false;
  c->rep_sync_due = c->ix.rep.depth != 0;
  if (new_entries) *new_entries = nn;
}

}  // namespace

extern "C" {

int skv_commit(skv_ctx* c, uint64_t* new_entries) {
  NvtxRange nvtx_range("skv_commit");
  if (!c) return SKV_ERR_ARG;
  return guard(c, [&] {
    check_usable(c);
    if (!c->pending)
      throw StateError(c->dropped_by_evict ? "skv_commit: the admitted batch was dropped by skv_evict (admit it again)"
                                           : "skv_commit without a preceding skv_admit");
    CK(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    if (c->p_n == 0) {
      release_slot(c);
      c->pending = false;
      c->rep_sync_due = c->ix.rep.depth != 0;  // an empty share still takes part in the merge
      if (new_entries) *new_entries = 0;
      return SKV_OK;
    }
    if (c->entries + c->tombstones + c->p_blocks > c->ix.cap - c->ix.cap / 8)
      throw CapacityError("index capacity exhausted (enable eviction: skv_enable_eviction / skv_set_tier_budget)");
    if (c->budget_on) {
      CK(cudaEventRecord(c->ev[5], s));
      const uint64_t before = c->entries + c->tombstones;
      const uint64_t made0 = c->node_next;
      ++c->batch_id;
      commit_budgeted(c);
      CK(cudaEventRecord(c->ev[6], s));
      sync_check(s);
      c->times.commit_ms = elapsed(c->ev[5], c->ev[6]);
      c->times.new_blocks = c->node_next - made0;
      (void)before;
      release_slot(c);
      c->pending = false;
      if (new_entries) *new_entries = c->times.new_blocks;
      return SKV_OK;
    }
    const CommitRun run = commit_enqueue(c);
    sync_check(s);  // the commit's one synchronisation (plus the rare ordered replay)
    commit_finish(c, run, new_entries);
    return SKV_OK;
  });
}

}  // extern "C"

namespace {

// advance_epoch + epoch_pass + roll (monitor.hpp:85-99, cache_index.hpp:296-299), enqueued: the
// host state (epoch, current window) advances in epoch_finish.  speculative: the pass aborts on
// the device, before touching anything, when the commit queued ahead of it raised an error or
// needs the ordered replay (counters[5] | counters[8]) -- the caller then runs it again.
struct EpochRun {
  uint64_t epoch;
  size_t pre;
  bool split;
};

EpochRun epoch_enqueue(skv_ctx* c, bool speculative) {
  cudaStream_t s = c->stream;
  const uint64_t epoch = c->epoch + 1;
  const uint32_t stamp = static_cast<uint32_t>(epoch);
  // grids cover the window lists' capacity; the kernels read the list lengths on the
  // device, so the epoch needs no host round trip before its kernels
  const int cur = c->cur, prev = 1 - c->cur;
  const uint32_t bound = 2 * c->pool_cap;
  // the pass as six kernels over the window lists' capacity (every entry its own thread) when the
  // last admit's window was large: the fused pass's co-resident grid strides over such lists with
  // less memory parallelism (config 4, ~0.5 M touched entries: 0.35 vs 0.29 ms); one cooperative
  // launch otherwise (small windows are launch-bound).  SKV_EPOCH_SPLIT=1 / 0 forces either.
  static const char* split_env = std::getenv("SKV_EPOCH_SPLIT");
  const bool split = split_env ? std::atoi(split_env) != 0 : c->touched_est > kEpochSplitMin;
  const uint32_t* guard = speculative ? c->counters : nullptr;
  const size_t pre = std::min<size_t>(kEpochEvPre, 2ull * c->pool_cap);
  const bool graphed = c->graphs && !split;
  auto issue = [&] {
    rec_ev(c, c->ev[8], s);
    CK(cudaMemsetAsync(c->counters + 3, 0, 8, s));  // n_cands, n_events
    if (!split) {
      // a graph's pass takes its stamps and arming from the device step state
      CK(skv::launch_epoch_fused(c->ix, c->touched, c->counters + 1, cur, stamp, c->cfg.entropy_jump,
                                 c->cfg.u_pre_max, c->cands, c->counters + 3, epoch, c->events, c->counters + 4,
                                 c->fired, c->counters, graphed ? c->dstate : nullptr,
                                 (graphed || speculative) ? c->counters : nullptr, c->device, s));
    } else {
      skv::launch_epoch_candidates(c->ix, c->touched[cur], c->counters + 1 + cur, c->pool_cap, 0, stamp,
                                   c->cfg.entropy_jump, c->cfg.u_pre_max, c->cands, c->counters + 3, s, guard);
      skv::launch_epoch_candidates(c->ix, c->touched[prev], c->counters + 1 + prev, c->pool_cap, 1, stamp,
                                   c->cfg.entropy_jump, c->cfg.u_pre_max, c->cands, c->counters + 3, s, guard);
      skv::launch_epoch_fire(c->ix, c->cands, c->counters + 3, bound, stamp, epoch, c->events, c->counters + 4,
                             c->fired, s, guard);
      skv::launch_epoch_propagate(c->ix, c->fired, c->counters + 4, bound, s, guard);
      skv::launch_epoch_roll(c->ix, c->touched[prev], c->counters + 1 + prev, c->pool_cap, 1, s, guard);
      skv::launch_epoch_roll(c->ix, c->touched[cur], c->counters + 1 + cur, c->pool_cap, 0, s, guard);
      // swap windows: the current list becomes the previous one (its count stays where it
      // is); the pool and the new current list start empty (the fused pass resets them itself)
      skv::launch_epoch_reset(c->counters, c->counters + 1 + prev, guard, s);
    }
    CK(cudaMemcpyAsync(c->host_small + kEpochCountSlot, c->counters + 4, 4, cudaMemcpyDeviceToHost, s));
    // the first events ride along with their count (events are rare: one synchronisation)
    CK(cudaMemcpyAsync(c->host_events, c->events, pre * sizeof(skv_event), cudaMemcpyDeviceToHost, s));
    rec_ev(c, c->ev[9], s);
  };
  if (graphed) {
    put_state(c, 2, c->rec_batch, epoch, speculative);
    run_graph(c, c->g_epoch, {reinterpret_cast<uintptr_t>(c->events), c->pool_cap}, issue);
  } else {
    issue();
  }
  return EpochRun{epoch, pre, split};
}

// After the synchronisation of a pass that ran: its events, and the host state advances.
void epoch_finish(skv_ctx* c, const EpochRun& run, skv_event* events, size_t cap, size_t* n_events,
                  uint64_t* epoch_out) {
  cudaStream_t s = c->stream;
  const uint32_t ne = c->host_small[kEpochCountSlot];
  std::vector<skv_event> ev(ne);
  if (ne <= run.pre) {
    std::copy(c->host_events, c->host_events + ne, ev.begin());
  } else {
    CK(cudaMemcpyAsync(ev.data(), c->events, ne * sizeof(skv_event), cudaMemcpyDeviceToHost, s));
    sync_check(s);
  }
  c->epoch = run.epoch;  // advance_epoch
  c->cur = 1 - c->cur;
  c->wstart = c->rec_batch + 1;  // user-set stamps of the closed window become stale
  c->times.epoch_ms = elapsed(c->ev[8], c->ev[9]);
  c->times.kernels_launched += run.split ? 7 : 1;
  std::sort(ev.begin(), ev.end(), [](const skv_event& x, const skv_event& y) {
    return x.h != y.h ? x.h < y.h : x.d < y.d;
  });
  if (events)
    for (size_t i = 0; i < ev.size() && i < cap; ++i) events[i] = ev[i];
  if (n_events) *n_events = ev.size();
  c->last_events = std::move(ev);  // the whole list stays retrievable (skv_last_events)
  if (epoch_out) *epoch_out = run.epoch;
}

}  // namespace

extern "C" {

int skv_epoch(skv_ctx* c, skv_event* events, size_t cap, size_t* n_events, uint64_t* epoch_out) {
  NvtxRange nvtx_range("skv_epoch");
  if (!c) return SKV_ERR_ARG;
  return guard(c, [&] {
    check_usable(c);
    CK(cudaSetDevice(c->device));
    ensure_admit_resolved(c);
    flush_record(c);
    const EpochRun run = epoch_enqueue(c, false);
    sync_check(c->stream);
    epoch_finish(c, run, events, cap, n_events, epoch_out);
    return SKV_OK;
  });
}

// admit + commit + epoch of one batch with one synchronisation in the common case: the epoch is
// queued behind the commit speculatively (it aborts itself on the device if the commit failed or
// needs the ordered replay; the epoch then runs again after the replay).  A small batch's step is
// bound by host round trips otherwise.
int skv_step(skv_ctx* c, const skv_batch* b, skv_admit_out* out, const skv_batch* prefetch_next,
             const skv_batch* stage_after, uint64_t* new_entries, skv_event* events, size_t cap, size_t* n_events,
             uint64_t* epoch_out) {
  NvtxRange nvtx_range("skv_step");
  if (!c || !b) return SKV_ERR_ARG;
  const bool fused = !c->budget_on && !c->evict_on && !c->ix.rep.depth;
  c->lazy_outputs = fused;  // the admit's output copies complete with the step's one synchronisation
  int rc = skv_admit(c, b, out);
  c->lazy_outputs = false;
  if (rc != SKV_OK) return rc;
  if (prefetch_next && (rc = skv_prefetch(c, prefetch_next)) != SKV_OK) {
    // the admitted batch stays pending: its outputs land now, not at a later commit (the caller
    // may drop `out` after this error)
    guard(c, [&] {
      ensure_admit_resolved(c);
      return SKV_OK;
    });
    return rc;
  }
  if (!fused || c->p_n == 0) {
    if ((rc = skv_commit(c, new_entries)) != SKV_OK) return rc;
    if (stage_after && (rc = skv_stage(c, stage_after)) != SKV_OK) return rc;
    return skv_epoch(c, events, cap, n_events, epoch_out);
  }
  return guard(c, [&]() -> int {
    if (c->entries + c->tombstones + c->p_blocks > c->ix.cap - c->ix.cap / 8)
      throw CapacityError("index capacity exhausted (enable eviction: skv_enable_eviction / skv_set_tier_budget)");
    const CommitRun crun = commit_enqueue(c);
    const EpochRun erun = epoch_enqueue(c, true);
    sync_check(c->stream);
    const bool epoch_ran = c->host_small[4] == 0 && c->host_small[5] == 0;  // the pass's own abort test
    commit_finish(c, crun, new_entries);  // raises the commit's errors; runs the ordered replay
    if (stage_after) {  // the committed batch's staging slot is free again: queue the H2D of a later batch
      const int rs = skv_stage(c, stage_after);
      if (rs != SKV_OK) return rs;
    }
    if (epoch_ran) {
      epoch_finish(c, erun, events, cap, n_events, epoch_out);
    } else {
      const EpochRun again = epoch_enqueue(c, false);
      sync_check(c->stream);
      epoch_finish(c, again, events, cap, n_events, epoch_out);
    }
    return SKV_OK;
  });
}

int skv_last_events(skv_ctx* c, skv_event* events, size_t cap, size_t* n_events) {
  if (!c || (cap && !events)) return SKV_ERR_ARG;
  for (size_t i = 0; i < c->last_events.size() && i < cap; ++i) events[i] = c->last_events[i];
  if (n_events) *n_events = c->last_events.size();
  return SKV_OK;
}

int skv_set_monitor_config(skv_ctx* c, double entropy_jump, uint64_t u_pre_max) {
  if (!c) return SKV_ERR_ARG;
  c->cfg.entropy_jump = entropy_jump;
  c->cfg.u_pre_max = u_pre_max;
  return SKV_OK;
}

int skv_set_label_policy(skv_ctx* c, int pending) {
  if (!c) return SKV_ERR_ARG;
  c->pending_labels = pending != 0;
  return SKV_OK;
}

int skv_resolve_blocks(skv_ctx* c, const uint64_t* h, const uint64_t* d, const uint32_t* block_offsets,
                       uint32_t n_prompts, const uint32_t* first_block, const uint8_t* labels) {
  if (!c || !block_offsets || (n_prompts && (!first_block || !labels))) return SKV_ERR_ARG;
  const size_t n = block_offsets[n_prompts];
  if (n && (!h || !d)) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    if (n_prompts == 0) return SKV_OK;
    if (block_offsets[0] != 0) throw ArgError("block_offsets must start at 0");
    for (uint32_t p = 0; p < n_prompts; ++p) {
      if (labels[p] != SKV_LABEL_PUBLIC && labels[p] != SKV_LABEL_PRIVATE && labels[p] != SKV_LABEL_RESTRICTED)
        throw ArgError("resolve: labels must be Private, Public or Restricted");
      if (first_block[p] > block_offsets[p + 1] - block_offsets[p]) throw ArgError("resolve: first_block past prompt");
    }
    ensure_admit_resolved(c);
    std::vector<void*> tmp;
    uint64_t* dh = dalloc<uint64_t>(std::max<size_t>(n, 1), tmp);
    uint64_t* dd = dalloc<uint64_t>(std::max<size_t>(n, 1), tmp);
    uint32_t* db = dalloc<uint32_t>(n_prompts + 1ull, tmp);
    uint32_t* df = dalloc<uint32_t>(n_prompts, tmp);
    uint8_t* dl = dalloc<uint8_t>(n_prompts, tmp);
    uint32_t* miss = dalloc<uint32_t>(1, tmp);
    cudaStream_t s = c->stream;
    if (n) CK(cudaMemcpyAsync(dh, h, n * 8, cudaMemcpyHostToDevice, s));
    if (n) CK(cudaMemcpyAsync(dd, d, n * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(db, block_offsets, (n_prompts + 1ull) * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(df, first_block, n_prompts * 4ull, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dl, labels, n_prompts, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(miss, 0, 4, s));
    skv::launch_resolve(c->ix, dh, dd, db, n_prompts, df, dl, static_cast<uint32_t>(n), miss, s);
    CK(cudaMemcpyAsync(c->host_small + 24, miss, 4, cudaMemcpyDeviceToHost, s));
    sync_check(s);
    for (void* q : tmp) cudaFree(q);
    if (c->host_small[24]) throw ArgError("resolve: a block of a classification span is not in the index");
    return SKV_OK;
  });
}

int skv_set_tiers(skv_ctx* c, const uint64_t* h, const uint64_t* d, const uint32_t* block_offsets, uint32_t n_prompts,
                  const uint8_t* tiers) {
  if (!c || !block_offsets) return SKV_ERR_ARG;
  const size_t n = block_offsets[n_prompts];
  if (n && (!h || !d || !tiers)) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    if (n == 0) return SKV_OK;
    if (block_offsets[0] != 0) throw ArgError("block_offsets must start at 0");
    std::vector<void*> tmp;
    uint64_t* dh = dalloc<uint64_t>(n, tmp);
    uint64_t* dd = dalloc<uint64_t>(n, tmp);
    uint8_t* dt = dalloc<uint8_t>(n, tmp);
    uint32_t* db = dalloc<uint32_t>(n_prompts + 1ull, tmp);
    cudaStream_t s = c->stream;
    CK(cudaMemcpyAsync(dh, h, n * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dd, d, n * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dt, tiers, n, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(db, block_offsets, (n_prompts + 1ull) * 4, cudaMemcpyHostToDevice, s));
    skv::launch_set_tiers(c->ix, dh, dd, db, n_prompts, dt, static_cast<uint32_t>(n), s);
    if (c->budget_on) {  // tier moves are accounted (not capacity-checked): recount the live entries
      auto* cnt = dalloc<unsigned long long>(3, tmp);
      skv::launch_count_tiers(c->ix, cnt, s);
      CK(cudaMemcpyAsync(c->host_small, cnt, 24, cudaMemcpyDeviceToHost, s));
      sync_check(s);
      std::memcpy(c->bud_used, c->host_small, 24);
    }
    sync_check(s);
    for (void* p : tmp) cudaFree(p);
    return SKV_OK;
  });
}

int skv_export(skv_ctx* c, skv_entry* out, size_t cap, size_t* n) {
  if (!c) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    ensure_admit_resolved(c);
    flush_record(c);
    std::vector<void*> tmp;
    cudaStream_t s = c->stream;
    uint32_t* dn = dalloc<uint32_t>(1, tmp);
    uint64_t room = std::max<uint64_t>(c->entries, 1);
    skv_entry* dout = nullptr;
    uint32_t cnt = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {  // the device count is exact even past the buffer
      dout = dalloc<skv_entry>(room, tmp);
      CK(cudaMemsetAsync(dout, 0, room * sizeof(skv_entry), s));  // defined struct padding
      CK(cudaMemsetAsync(dn, 0, 4, s));
      skv::launch_export(c->ix, c->users_tab.rev, dout, dn, static_cast<uint32_t>(room), s);
      CK(cudaMemcpyAsync(&cnt, dn, 4, cudaMemcpyDeviceToHost, s));
      sync_check(s);
      if (cnt <= room) break;
      room = cnt;
    }
    if (out && cnt) CK(cudaMemcpy(out, dout, std::min<size_t>(cnt, cap) * sizeof(skv_entry), cudaMemcpyDeviceToHost));
    for (void* p : tmp) cudaFree(p);
    if (n) *n = cnt;
    return SKV_OK;
  });
}

uint64_t skv_entry_count(skv_ctx* c) { return c ? c->entries : 0; }

int skv_enable_eviction(skv_ctx* c, int tiered_demotion) {
  if (!c) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    if (c->evict_on) return SKV_OK;
    if (c->entries || c->batch_id) throw StateError("skv_enable_eviction must precede the first admit");
    if (c->ix.rep.depth) throw StateError("the replicated layer and eviction cannot be combined");
    skv::EvictMeta* em = dalloc<skv::EvictMeta>(c->ix.cap, c->owned);
    CK(cudaMemsetAsync(em, 0, c->ix.cap * sizeof(skv::EvictMeta), c->stream));
    const uint64_t N = std::max<uint64_t>(c->max_prompts, 1);
    c->ev_counts = dalloc<uint32_t>(N, c->owned);
    c->ev_incl = dalloc<uint32_t>(N, c->owned);
    c->ev_temp_bytes = skv::evict_temp_bytes(static_cast<uint32_t>(N), c->ix.cap);
    c->ev_temp = dalloc<uint8_t>(c->ev_temp_bytes, c->owned);
    sync_check(c->stream);
    c->ix.em = em;
    c->evict_on = true;
    c->evict_tiered = tiered_demotion != 0;
    return SKV_OK;
  });
}

int skv_set_tier_budget(skv_ctx* c, uint64_t hbm_blocks, uint64_t dram_blocks, uint64_t ssd_blocks) {
  if (!c) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    if (!c->evict_on) throw StateError("skv_set_tier_budget needs eviction (skv_enable_eviction first)");
    if (c->entries || c->batch_id || c->pending) throw StateError("skv_set_tier_budget must precede the first admit");
    if (!c->budget_on) {
      c->vstamp = dalloc<uint32_t>(c->ix.cap, c->owned);
      CK(cudaMemsetAsync(c->vstamp, 0xff, c->ix.cap * 4, c->stream));
      c->mark_cap = static_cast<uint32_t>(std::min<uint64_t>(c->max_blocks + 1, 0xffffffffull));
      c->mark_list = dalloc<uint32_t>(c->mark_cap, c->owned);
      c->n_mark = dalloc<uint32_t>(1, c->owned);
      uint64_t dc = 1024;
      while (dc < 2 * c->max_blocks) dc <<= 1;
      c->dry_cap = dc;
      c->dry_tab = dalloc<ulonglong2>(dc, c->owned);
      c->dry_minp = dalloc<uint32_t>(dc, c->owned);
      c->dry_slot = dalloc<uint32_t>(c->max_blocks + 1, c->owned);
      c->needed = dalloc<uint32_t>(c->max_prompts + 1, c->owned);
      c->sim = dalloc<skv::BudgetSim>(1, c->owned);
      c->nb_dev = dalloc<unsigned long long>(1, c->owned);
      if (!c->ev_eff) {
        c->ev_eff = dalloc<unsigned long long>(c->ix.cap, c->owned);
        c->ev_n = dalloc<uint32_t>(1, c->owned);
      }
      sync_check(c->stream);
    }
    c->bud_cap[0] = hbm_blocks;
    c->bud_cap[1] = dram_blocks;
    c->bud_cap[2] = ssd_blocks;
    c->budget_on = true;
    return SKV_OK;
  });
}

int skv_tier_usage(skv_ctx* c, uint64_t* used3, uint64_t* cap3) {
  if (!c) return SKV_ERR_ARG;
  for (int t = 0; t < 3; ++t) {
    if (used3) used3[t] = c->bud_used[t];
    if (cap3) cap3[t] = c->bud_cap[t];
  }
  return SKV_OK;
}

int skv_last_drops(skv_ctx* c, uint32_t* prompts, size_t cap, size_t* n) {
  if (!c || !n) return SKV_ERR_ARG;
  *n = c->dropped.size();
  if (prompts)
    for (size_t i = 0; i < c->dropped.size() && i < cap; ++i) prompts[i] = c->dropped[i];
  return SKV_OK;
}

int skv_evict(skv_ctx* c, uint64_t needed_blocks, uint64_t epoch, uint64_t* n_evicted, uint64_t* victims_h,
              uint64_t* victims_d, size_t cap) {
  NvtxRange nvtx_range("skv_evict");
  (void)epoch;  // the victim order only compares access epochs (epoch - access_epoch, cache_index.hpp:709)
  if (!c || !n_evicted) return SKV_ERR_ARG;
  *n_evicted = 0;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    if (!c->evict_on) throw StateError("eviction is not enabled (skv_enable_eviction before the first admit)");
    if (needed_blocks == 0) throw ArgError("evict: needed must be positive");
    check_usable(c);
    // an admitted, uncommitted batch is dropped: its lookups ran (and its monitor records were
    // applied by flush_record), but its commit would attach new blocks to entries this call may
    // tombstone (the reference pins a request's path around insert, cache_index.hpp:347-356,
    // serving_sim.hpp:196,215), so a later skv_commit raises SKV_ERR_STATE
    if (c->pending && c->p_n) c->dropped_by_evict = true;
    c->pending = false;
    ensure_admit_resolved(c);
    flush_record(c);
    release_slot(c);
    cudaStream_t s = c->stream;
    if (!c->ev_eff) {  // per-slot effective keys, on first use
      c->ev_eff = dalloc<unsigned long long>(c->ix.cap, c->owned);
      c->ev_n = dalloc<uint32_t>(1, c->owned);
    }
    // candidate lists sized by the live entries of this call (40 B each), freed after
    std::vector<void*> tmp;
    const uint64_t L = std::max<uint64_t>(c->entries, 1);
    auto* keys_a = dalloc<unsigned long long>(L, tmp);
    auto* keys_b = dalloc<unsigned long long>(L, tmp);
    auto* vals_a = dalloc<uint32_t>(L, tmp);
    auto* vals_b = dalloc<uint32_t>(L, tmp);
    auto* vh = dalloc<uint64_t>(L, tmp);
    auto* vd = dalloc<uint64_t>(L, tmp);
    if (c->budget_on && c->evict_tiered) {  // evict_or_demote with bounded DRAM / SSD (cascade)
      for (void* p : tmp) cudaFree(p);
      tmp.clear();
      const TieredOutcome o = run_tiered(c, nullptr, nullptr, 0, 0, needed_blocks, 0);
      c->entries -= o.freed;
      c->tombstones += o.freed;
      for (int t = 0; t < 3; ++t) c->bud_used[t] = o.used[t];
      *n_evicted = o.hbm_out;
      if (o.r.dropped == 0) throw CapacityError("evict: no unpinned candidate leaf");
      return SKV_OK;
    }
    const uint32_t v = skv::launch_evict(c->ix, needed_blocks, c->ev_eff, keys_a, keys_b, vals_a, vals_b, c->ev_n,
                                         c->ev_temp, c->ev_temp_bytes, vh, vd, c->host_small,
                                         c->evict_tiered ? 1 : 0, s);
    const size_t k = std::min<size_t>(v, cap);
    if (victims_h && k) CK(cudaMemcpyAsync(victims_h, vh, k * 8, cudaMemcpyDeviceToHost, s));
    if (victims_d && k) CK(cudaMemcpyAsync(victims_d, vd, k * 8, cudaMemcpyDeviceToHost, s));
    sync_check(s);
    for (void* p : tmp) cudaFree(p);
    if (!c->evict_tiered) {
      c->entries -= v;
      c->tombstones += v;
      c->bud_used[0] -= std::min<uint64_t>(c->bud_used[0], v);
    } else {  // unbounded lower tiers: victims move HBM -> DRAM
      c->bud_used[0] -= std::min<uint64_t>(c->bud_used[0], v);
      c->bud_used[1] += v;
    }
    *n_evicted = v;
    if (v < needed_blocks) throw CapacityError("evict: no unpinned candidate leaf");
    return SKV_OK;
  });
}

// ------------------------------------------------------------------ replicated layer
int skv_set_replicated_depth(skv_ctx* c, uint32_t depth) {
  if (!c) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    if (c->entries || c->batch_id || c->pending) throw StateError("skv_set_replicated_depth must precede the first admit");
    if (c->evict_on) throw StateError("the replicated layer and eviction cannot be combined");
    if (depth == 0 || c->ix.rep.depth) {
      if (depth != c->ix.rep.depth && c->ix.rep.depth) throw StateError("replicated depth already set");
      return SKV_OK;
    }
    skv::RepLayer& R = c->ix.rep;
    uint32_t pairs = 1u << 16;
    while (pairs < 4 * c->cfg.max_window_entries && pairs < (1u << 24)) pairs <<= 1;
    R.pair_key = dalloc<ulonglong2>(pairs, c->owned);
    R.pair_first = dalloc<uint32_t>(pairs, c->owned);
    R.pair_gid = dalloc<unsigned long long>(pairs, c->owned);
    skv::RepScratch& W = c->rep_w;
    W.gid_a = dalloc<unsigned long long>(pairs, c->owned);
    W.gid_b = dalloc<unsigned long long>(pairs, c->owned);
    W.val_a = dalloc<uint32_t>(pairs, c->owned);
    W.val_b = dalloc<uint32_t>(pairs, c->owned);
    W.slot_a = dalloc<uint32_t>(pairs, c->owned);
    W.slot_b = dalloc<uint32_t>(pairs, c->owned);
    W.n = dalloc<uint32_t>(1, c->owned);
    W.host_n = c->host_small + 40;
    W.temp_bytes = skv::rep_sort_temp_bytes(pairs);
    W.temp = dalloc<uint8_t>(W.temp_bytes, c->owned);
    R.pair_cnt = dalloc<uint32_t>(pairs, c->owned);
    R.pair_mask = pairs - 1;
    R.new_cap = static_cast<uint32_t>(std::min<uint64_t>(c->max_blocks, 1ull << 26));
    R.new_list = dalloc<uint32_t>(R.new_cap, c->owned);
    R.new_n = dalloc<uint32_t>(1, c->owned);
    R.err = dalloc<uint32_t>(1, c->owned);
    c->rep_ents = dalloc<skv_rep_entry>(R.new_cap, c->owned);
    c->rep_accs = dalloc<skv_rep_access>(pairs, c->owned);
    c->rep_gids = dalloc<uint64_t>(c->max_prompts, c->owned);
    CK(cudaMemsetAsync(R.new_n, 0, 4, c->stream));
    CK(cudaMemsetAsync(R.err, 0, 4, c->stream));
    R.depth = depth;
    skv::launch_rep_clear(c->ix, c->stream);
    sync_check(c->stream);
    return SKV_OK;
  });
}

int skv_replica_export(skv_ctx* c, const uint64_t* gids, skv_rep_entry* ents, size_t ecap, size_t* n_ents,
                       skv_rep_access* accs, size_t acap, size_t* n_accs, int accs_on_device) {
  NvtxRange nvtx_range("skv_replica_export");
  if (!c || !n_ents || !n_accs) return SKV_ERR_ARG;
  *n_ents = *n_accs = 0;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    if (!c->ix.rep.depth) throw StateError("no replicated layer (skv_set_replicated_depth)");
    if (!c->rep_sync_due) throw StateError("skv_replica_export: no committed batch to export");
    if (c->p_n && !gids) throw ArgError("prompt_gids required");
    cudaStream_t s = c->stream;
    if (c->p_n) CK(cudaMemcpyAsync(c->rep_gids, gids, c->p_n * 8ull, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(c->host_small + 32, c->ix.rep.new_n, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(c->host_small + 33, c->ix.rep.err, 4, cudaMemcpyDeviceToHost, s));
    sync_check(s);
    if (c->host_small[33]) throw CapacityError("replicated layer: pair table or new-entry list full");
    const uint32_t nn = std::min(c->host_small[32], c->ix.rep.new_cap);
    CK(cudaMemsetAsync(c->counters + 13, 0, 4, s));
    skv::launch_rep_export(c->ix, c->users_tab.rev, c->rep_gids, nn, c->rep_ents, c->rep_accs, c->counters + 13,
                           c->ix.rep.pair_mask + 1, s);
    CK(cudaMemcpyAsync(c->host_small + 34, c->counters + 13, 4, cudaMemcpyDeviceToHost, s));
    sync_check(s);
    const uint32_t na = c->host_small[34];
    *n_ents = nn;
    *n_accs = na;
    if (nn > ecap || na > acap || (nn && !ents) || (na && !accs))
      throw CapacityError("skv_replica_export: buffers too small (sizes returned)");
    if (nn) CK(cudaMemcpyAsync(ents, c->rep_ents, nn * sizeof(skv_rep_entry), cudaMemcpyDeviceToHost, s));
    if (na)
      CK(cudaMemcpyAsync(accs, c->rep_accs, na * sizeof(skv_rep_access),
                         accs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    sync_check(s);
    return SKV_OK;
  });
}

int skv_replica_apply(skv_ctx* c, const skv_rep_entry* ents, size_t n_ents, const skv_rep_access* accs,
                      size_t n_accs, int accs_on_device) {
  NvtxRange nvtx_range("skv_replica_apply");
  if (!c || (n_ents && !ents) || (n_accs && !accs)) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    if (!c->ix.rep.depth) throw StateError("no replicated layer (skv_set_replicated_depth)");
    if (!c->rep_sync_due) throw StateError("skv_replica_apply: no committed batch to apply to");
    cudaStream_t s = c->stream;
    const size_t off_a = (n_ents * sizeof(skv_rep_entry) + 15) & ~size_t(15);
    const size_t off_c = (off_a + n_accs * sizeof(skv_rep_access) + 15) & ~size_t(15);
    const size_t need = off_c + n_ents * 8 + 64;
    if (need > c->rep_in_bytes) {
      if (c->rep_in) CK(cudaFree(c->rep_in));
      c->rep_in_bytes = need * 2;
      CK(cudaMalloc(&c->rep_in, c->rep_in_bytes));
    }
    if (n_ents > c->rep_in_ents) {
      if (c->rep_slots) CK(cudaFree(c->rep_slots));
      if (c->rep_uidx) CK(cudaFree(c->rep_uidx));
      c->rep_in_ents = n_ents * 2;
      CK(cudaMalloc(&c->rep_slots, c->rep_in_ents * 4));
      CK(cudaMalloc(&c->rep_uidx, c->rep_in_ents * 4));
    }
    auto* dents = static_cast<skv_rep_entry*>(c->rep_in);
    auto* daccs = reinterpret_cast<skv_rep_access*>(static_cast<uint8_t*>(c->rep_in) + off_a);
    auto* dcr = reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(c->rep_in) + off_c);
    if (n_ents) CK(cudaMemcpyAsync(dents, ents, n_ents * sizeof(skv_rep_entry), cudaMemcpyHostToDevice, s));
    if (n_accs && !accs_on_device)
      CK(cudaMemcpyAsync(daccs, accs, n_accs * sizeof(skv_rep_access), cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(c->counters + 14, 0, 4, s));  // entries claimed here
    CK(cudaMemsetAsync(c->ix.rep.err, 0, 4, s));
    if (n_ents) {  // creators: interned like an admitted prompt's user
      static_assert(offsetof(skv_rep_entry, creator) % 8 == 0, "");
      std::vector<uint64_t> cr(n_ents);
      for (size_t i = 0; i < n_ents; ++i) cr[i] = ents[i].creator;
      CK(cudaMemcpyAsync(dcr, cr.data(), n_ents * 8, cudaMemcpyHostToDevice, s));
      skv::launch_intern_users(c->users_tab, dcr, static_cast<uint32_t>(n_ents), c->rep_uidx, c->counters + 5, s);
    }
    skv::MonCtx m;
    m.hdr = c->set_hdr;
    m.tab = c->set_tab;
    m.pool_cap = c->pool_cap;
    m.pool_count = c->counters + 0;
    m.touched = c->touched[c->cur];
    m.n_touched = c->counters + 1 + c->cur;
    m.batch = c->rec_batch;  // the batch whose accesses these are
    m.wstart = c->wstart;
    m.err = c->counters + 5;
    m.matched_total = c->counters + 10;
    if (n_accs > c->ix.rep.pair_mask + 1ull) throw CapacityError("skv_replica_apply: more accesses than the pair table");
    skv::launch_rep_clear(c->ix, s);  // the local aggregation was exported: the table merges now
    skv::launch_rep_apply(c->ix, m, dents, c->rep_uidx, static_cast<uint32_t>(n_ents), c->rep_slots, c->counters + 14,
                          accs_on_device ? static_cast<const void*>(accs) : daccs, static_cast<uint32_t>(n_accs),
                          c->rep_w, c->ix.rep.err, s);
    skv::launch_rep_clear(c->ix, s);
    CK(cudaMemsetAsync(c->ix.rep.new_n, 0, 4, s));
    CK(cudaMemcpyAsync(c->host_small + 35, c->counters + 14, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(c->host_small + 36, c->ix.rep.err, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(c->host_small + 37, c->counters + 5, 4, cudaMemcpyDeviceToHost, s));
    sync_check(s);
    c->entries += c->host_small[35];
    c->rep_sync_due = false;
    if (c->host_small[36] || (c->host_small[37] & 9u)) {
      c->poisoned = "replicated-layer apply failed (an entry, a parent or an accessed key is missing, or a pool is full)";
      throw CapacityError(c->poisoned);
    }
    return SKV_OK;
  });
}

// ------------------------------------------------------------------ per-call facade entry points
int skv_lookup(skv_ctx* c, const skv_batch* b, skv_admit_out* out) {
  if (!c || !b) return SKV_ERR_ARG;
  if (c->ix.rep.depth) return fail(c, SKV_ERR_STATE, "skv_lookup: not with a replicated layer");
  c->no_record = true;
  const int rc = skv_admit(c, b, out);
  c->no_record = false;
  if (rc == SKV_OK) c->pending = false;  // nothing to commit, nothing recorded
  return rc;
}

int skv_insert(skv_ctx* c, const skv_batch* b, uint64_t* new_entries) {
  if (!c || !b) return SKV_ERR_ARG;
  if (c->ix.rep.depth) return fail(c, SKV_ERR_STATE, "skv_insert: not with a replicated layer");
  c->no_record = true;
  int rc = skv_admit(c, b, nullptr);
  c->no_record = false;
  if (rc != SKV_OK) return rc;
  return skv_commit(c, new_entries);
}

namespace {
// device slots of host keys (SKV_ERR_ARG when one is not a live entry)
std::vector<void*> find_slots(skv_ctx* c, const uint64_t* h, const uint64_t* d, size_t n, uint32_t** slots) {
  std::vector<void*> tmp;
  uint64_t* dh = dalloc<uint64_t>(n, tmp);
  uint64_t* dd = dalloc<uint64_t>(n, tmp);
  *slots = dalloc<uint32_t>(n, tmp);
  cudaStream_t s = c->stream;
  CK(cudaMemcpyAsync(dh, h, n * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dd, d, n * 8, cudaMemcpyHostToDevice, s));
  skv::launch_find_entries(c->ix, dh, dd, static_cast<uint32_t>(n), *slots, s);
  std::vector<uint32_t> hs(n);
  CK(cudaMemcpyAsync(hs.data(), *slots, n * 4, cudaMemcpyDeviceToHost, s));
  sync_check(s);
  for (uint32_t v : hs)
    if (v == skv::kNone) {
      for (void* q : tmp) cudaFree(q);
      throw ArgError("no such entry");
    }
  return tmp;
}

skv::MonCtx current_window(skv_ctx* c) {
  skv::MonCtx m;
  m.hdr = c->set_hdr;
  m.tab = c->set_tab;
  m.pool_cap = c->pool_cap;
  m.pool_count = c->counters + 0;
  m.touched = c->touched[c->cur];
  m.n_touched = c->counters + 1 + c->cur;
  m.batch = c->rec_batch;
  m.wstart = c->wstart;
  m.err = c->counters + 5;
  m.matched_total = c->counters + 10;
  return m;
}
}  // namespace

int skv_get_entries(skv_ctx* c, const uint64_t* h, const uint64_t* d, size_t n, skv_entry* out, uint8_t* found) {
  if (!c || (n && (!h || !d || !out))) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    ensure_admit_resolved(c);
    flush_record(c);
    if (!n) return SKV_OK;
    std::vector<void*> tmp;
    uint64_t* dh = dalloc<uint64_t>(n, tmp);
    uint64_t* dd = dalloc<uint64_t>(n, tmp);
    uint32_t* sl = dalloc<uint32_t>(n, tmp);
    cudaStream_t s = c->stream;
    CK(cudaMemcpyAsync(dh, h, n * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dd, d, n * 8, cudaMemcpyHostToDevice, s));
    skv::launch_find_entries(c->ix, dh, dd, static_cast<uint32_t>(n), sl, s);
    std::vector<uint32_t> hs(n);
    CK(cudaMemcpyAsync(hs.data(), sl, n * 4, cudaMemcpyDeviceToHost, s));
    sync_check(s);
    std::vector<uint64_t> rev(1);
    for (size_t i = 0; i < n; ++i) {
      if (found) found[i] = hs[i] != skv::kNone;
      out[i] = skv_entry{};
      if (hs[i] == skv::kNone) continue;
      skv::Entry e;
      CK(cudaMemcpy(&e, c->ix.e + hs[i], sizeof(e), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(rev.data(), c->users_tab.rev + e.rec.creator, 8, cudaMemcpyDeviceToHost));
      out[i].h = e.rec.h;
      out[i].d = e.rec.d;
      out[i].creator = rev[0];
      out[i].label = static_cast<uint8_t>(skv::meta_label(e.rec.meta));
      out[i].owner = static_cast<uint8_t>(skv::meta_owner(e.rec.meta));
      out[i].tier = static_cast<uint8_t>(skv::meta_tier(e.rec.meta));
      out[i].hit_cur = e.stats.hit_cur;
      out[i].u_cnt = e.stats.u_cnt;
      out[i].hit_pre = e.stats.hit_pre;
      out[i].u_pre = e.stats.u_pre;
    }
    for (void* q : tmp) cudaFree(q);
    return SKV_OK;
  });
}

int skv_label_entries(skv_ctx* c, const uint64_t* h, const uint64_t* d, size_t n, uint8_t label, int propagate,
                      size_t* changed) {
  if (!c || !n || !h || !d || label > SKV_LABEL_RESTRICTED) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    ensure_admit_resolved(c);
    uint32_t* sl = nullptr;
    std::vector<void*> tmp = find_slots(c, h, d, n, &sl);
    unsigned long long* ch = dalloc<unsigned long long>(1, tmp);
    // promotion to Public never propagates (cache_index.hpp:658-662)
    const int prop = propagate && (label == SKV_LABEL_PRIVATE || label == SKV_LABEL_RESTRICTED);
    skv::launch_label_entries(c->ix, sl, static_cast<uint32_t>(n), label, prop, ch, c->stream);
    unsigned long long hc = 0;
    CK(cudaMemcpyAsync(c->host_small + 44, ch, 8, cudaMemcpyDeviceToHost, c->stream));
    sync_check(c->stream);
    std::memcpy(&hc, c->host_small + 44, 8);
    for (void* q : tmp) cudaFree(q);
    if (changed) *changed = hc;
    return SKV_OK;
  });
}

int skv_record_accesses(skv_ctx* c, const uint64_t* h, const uint64_t* d, const uint64_t* users, size_t n) {
  if (!c || (n && (!h || !d || !users))) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    check_usable(c);
    ensure_admit_resolved(c);
    flush_record(c);
    if (!n) return SKV_OK;
    uint32_t* sl = nullptr;
    std::vector<void*> tmp = find_slots(c, h, d, n, &sl);
    uint64_t* du = dalloc<uint64_t>(n, tmp);
    CK(cudaMemcpyAsync(du, users, n * 8, cudaMemcpyHostToDevice, c->stream));
    skv::launch_record_list(c->ix, current_window(c), sl, du, static_cast<uint32_t>(n), c->stream);
    CK(cudaMemcpyAsync(c->host_small + 46, c->counters + 5, 4, cudaMemcpyDeviceToHost, c->stream));
    sync_check(c->stream);
    for (void* q : tmp) cudaFree(q);
    if (c->host_small[46] & 1u) throw CapacityError("monitor window user-set pool exhausted (raise max_window_entries)");
    return SKV_OK;
  });
}

int skv_roll_entries(skv_ctx* c, const uint64_t* h, const uint64_t* d, size_t n) {
  if (!c || (n && (!h || !d))) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    check_usable(c);
    ensure_admit_resolved(c);
    flush_record(c);
    if (!n) return SKV_OK;
    uint32_t* sl = nullptr;
    std::vector<void*> tmp = find_slots(c, h, d, n, &sl);
    skv::launch_roll_list(c->ix, current_window(c), sl, static_cast<uint32_t>(n), c->stream);
    sync_check(c->stream);
    for (void* q : tmp) cudaFree(q);
    return SKV_OK;
  });
}

int skv_check_anomaly(skv_ctx* c, uint64_t h, uint64_t d, uint64_t epoch, skv_event* ev, int* fired) {
  if (!c || !ev || !fired) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    check_usable(c);
    ensure_admit_resolved(c);
    flush_record(c);
    uint32_t* sl = nullptr;
    std::vector<void*> tmp = find_slots(c, &h, &d, 1, &sl);
    uint32_t slot = 0;
    CK(cudaMemcpy(&slot, sl, 4, cudaMemcpyDeviceToHost));
    skv_event* dev = dalloc<skv_event>(1, tmp);
    int* df = dalloc<int>(1, tmp);
    skv::launch_check_one(c->ix, slot, c->cfg.entropy_jump, c->cfg.u_pre_max, epoch, dev, df, c->stream);
    CK(cudaMemcpyAsync(ev, dev, sizeof(skv_event), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(fired, df, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    sync_check(c->stream);
    for (void* q : tmp) cudaFree(q);
    return SKV_OK;
  });
}

int skv_leak_flags(skv_ctx* c, const uint32_t* span_off, const uint64_t* span_begin, const uint64_t* span_end,
                   uint8_t* flags, uint64_t* n_leaks) {
  if (!c || !span_off) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    ensure_admit_resolved(c);
    const uint32_t N = c->last_n;
    if (span_off[0] != 0) throw ArgError("span offsets must start at 0");
    const size_t ns = span_off[N];
    if (ns && (!span_begin || !span_end)) throw ArgError("null span arrays");
    std::vector<void*> tmp;
    uint32_t* doff = dalloc<uint32_t>(N + 1ull, tmp);
    uint64_t* db = dalloc<uint64_t>(std::max<size_t>(ns, 1), tmp);
    uint64_t* de = dalloc<uint64_t>(std::max<size_t>(ns, 1), tmp);
    unsigned long long* dn = dalloc<unsigned long long>(1, tmp);
    uint8_t* df = flags ? dalloc<uint8_t>(std::max<uint64_t>(c->p_blocks, 1), tmp) : nullptr;
    cudaStream_t s = c->stream;
    CK(cudaMemcpyAsync(doff, span_off, (N + 1ull) * 4, cudaMemcpyHostToDevice, s));
    if (ns) CK(cudaMemcpyAsync(db, span_begin, ns * 8, cudaMemcpyHostToDevice, s));
    if (ns) CK(cudaMemcpyAsync(de, span_end, ns * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(dn, 0, 8, s));
    skv::launch_leak_flags(c->blk_off, c->blabel, doff, db, de, N, c->cfg.block_tokens, df, dn, s);
    unsigned long long hn = 0;
    CK(cudaMemcpyAsync(c->host_small + 48, dn, 8, cudaMemcpyDeviceToHost, s));
    if (flags && c->p_blocks) CK(cudaMemcpyAsync(flags, df, c->p_blocks, cudaMemcpyDeviceToHost, s));
    sync_check(s);
    std::memcpy(&hn, c->host_small + 48, 8);
    for (void* q : tmp) cudaFree(q);
    if (n_leaks) *n_leaks = hn;
    return SKV_OK;
  });
}

int skv_last_times(skv_ctx* c, skv_stage_times* out) {
  if (!c || !out) return SKV_ERR_ARG;
  return guard(c, [&] {
    ensure_admit_resolved(c);
    *out = c->times;
    return SKV_OK;
  });
}

int skv_tier1_scan(skv_ctx* c, const char* text, size_t len, uint32_t* mask) {
  if (!c || (!text && len) || !mask) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    std::vector<void*> tmp;
    uint8_t* dt = dalloc<uint8_t>(len + 1, tmp);
    const uint32_t words = c->mask_words;
    uint32_t* dm = dalloc<uint32_t>(words, tmp);
    cudaStream_t s = c->stream;
    if (len) CK(cudaMemcpyAsync(dt, text, len, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(dm, 0, 4ull * words, s));
    for (const auto& g : c->groups)
      skv::launch_scan_text(dt, static_cast<uint32_t>(len), g.dev, dm + g.word, g.shift, s);
    CK(cudaMemcpyAsync(mask, dm, 4ull * words, cudaMemcpyDeviceToHost, s));
    sync_check(s);
    for (void* p : tmp) cudaFree(p);
    return SKV_OK;
  });
}

int skv_tier1_scan_batch(skv_ctx* c, const char* text, const uint64_t* offsets, uint32_t n, uint32_t* rule_masks) {
  if (!c || !offsets || (n && !rule_masks)) return SKV_ERR_ARG;
  return guard(c, [&] {
    if (offsets[0] != 0) throw ArgError("offsets[0] must be 0");
    for (uint32_t i = 0; i < n; ++i)
      if (offsets[i + 1] < offsets[i]) throw ArgError("offsets must be non-decreasing");
    const uint64_t len = offsets[n];
    if (len && !text) throw ArgError("null text");
    if (n == 0) return SKV_OK;
    CK(cudaSetDevice(c->device));
    std::vector<void*> tmp;
    uint8_t* dt = dalloc<uint8_t>(len + 1, tmp);
    uint64_t* doff = dalloc<uint64_t>(n + 1ull, tmp);
    const uint64_t words = c->mask_words;
    uint32_t* dm = dalloc<uint32_t>(n * words, tmp);
    cudaStream_t s = c->stream;
    try {
      if (len) CK(cudaMemcpyAsync(dt, text, len, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(doff, offsets, (n + 1ull) * 8, cudaMemcpyHostToDevice, s));
      CK(cudaMemsetAsync(dm, 0, n * words * 4, s));
      for (const auto& g : c->groups) skv::launch_scan_texts(dt, doff, n, g.dev, dm + g.word * n, g.shift, s);
      CK(cudaMemcpyAsync(rule_masks, dm, n * words * 4, cudaMemcpyDeviceToHost, s));
      sync_check(s);
    } catch (...) {
      for (void* p : tmp) cudaFree(p);
      throw;
    }
    for (void* p : tmp) cudaFree(p);
    return SKV_OK;
  });
}

int skv_token_seq_digest(skv_ctx* c, const uint32_t* tokens, size_t n, uint64_t* digest) {
  if (!c || (!tokens && n) || !digest) return SKV_ERR_ARG;
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    std::vector<void*> tmp;
    uint32_t* dt = dalloc<uint32_t>(n + 1, tmp);
    uint64_t* dd = dalloc<uint64_t>(1, tmp);
    cudaStream_t s = c->stream;
    if (n) CK(cudaMemcpyAsync(dt, tokens, n * 4, cudaMemcpyHostToDevice, s));
    skv::launch_digest(dt, static_cast<uint32_t>(n), dd, s);
    CK(cudaMemcpyAsync(c->host_small, dd, 8, cudaMemcpyDeviceToHost, s));
    sync_check(s);
    std::memcpy(digest, c->host_small, 8);
    for (void* p : tmp) cudaFree(p);
    return SKV_OK;
  });
}

}  // extern "C"
