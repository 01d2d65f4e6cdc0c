// oracle/ref_harness.cpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// Thin extern "C" harness around the UNMODIFIED SafeKV reference headers, compiled
// read-only from /root/reference/proj/include by oracle/Makefile into
// oracle/_ref/libsafekv_ref.so.  It executes the parity contract of SURVEY.md
// Appendix A using reference code only:
//   * block digest      safekv::token_seq_digest            (core.hpp:68-73)
//   * chained key       safekv::Fnv1a64 update_u64 x2       (util.hpp:58-81)
//   * window verdicts   CompiledRuleSet::scan               (detection.hpp:148-170)
//                       on detokenize_bytes(window)          (core.hpp:114-119)
//   * lookup            RadixCacheIndex::match_prefix        (cache_index.hpp:213-237)
//                       over interned block-content ids (one node per block,
//                       ensure_boundary cache_index.hpp:400-418)
//   * record            EntropyMonitor::record_access        (monitor.hpp:50)
//   * commit            RadixCacheIndex::insert + set_label  (cache_index.hpp:152-205,312-315)
//   * epoch             advance_epoch + EntropyMonitor::epoch_pass (cache_index.hpp:296, monitor.hpp:85-99)
// plus safekv::generate (workload.hpp:428-700) for the config-1 golden fixture.
//
// Tests, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
// arm are the only callers.
#include <safekv/cache_index.hpp>
#include <safekv/core.hpp>
#include <safekv/detection.hpp>
#include <safekv/monitor.hpp>
#include <safekv/serving_sim.hpp>
#include <safekv/util.hpp>
#include <safekv/workload.hpp>

#include <atomic>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

using namespace safekv;

namespace {

void put_err(char* err, size_t cap, const std::string& msg) {
  if (!err || cap == 0) return;
  size_t n = std::min(cap - 1, msg.size());
  std::memcpy(err, msg.data(), n);
  err[n] = 0;
}

struct RulesBox {
  std::shared_ptr<const CompiledRuleSet> set;
};

// Bit i of the result = rule i (reference list order) matched and is enabled.
// Derived from the reference verdict: categories are recomputed per rule by
// scanning with single-rule snapshots would change semantics, so instead the
// harness compiles one single-rule snapshot per rule once (same flags) and ORs.
struct RuleMasks {
  std::vector<std::shared_ptr<const CompiledRuleSet>> single;  // one snapshot per rule
};

std::string content_key(const uint32_t* t, uint32_t n) {
  return std::string(reinterpret_cast<const char*>(t), static_cast<size_t>(n) * 4);
}

uint64_t block_digest(const uint32_t* t, uint32_t n) {
  TokenSeq s(t, t + n);
  return token_seq_digest(s);
}

uint64_t chain_key(uint64_t prev_h, uint64_t d) {
  Fnv1a64 f;
  f.update_u64(prev_h);
  f.update_u64(d);
  return f.digest();
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------- rules
void* ref_rules_default() {
  RuleEngine eng;
  auto* box = new RulesBox{eng.active()};
  return box;
}

void* ref_rules_load(const char* json, size_t len, char* err, size_t errcap) {
  try {
    RuleEngine eng;
    auto j = nlohmann::json::parse(std::string(json, len));
    auto set = eng.load_rules_json(j);
    return new RulesBox{set};
  } catch (const std::exception& e) {
    put_err(err, errcap, e.what());
    return nullptr;
  }
}

void ref_rules_free(void* r) { delete static_cast<RulesBox*>(r); }

uint32_t ref_rules_count(void* r) { return static_cast<uint32_t>(static_cast<RulesBox*>(r)->set->size()); }

// Reference verdict: sensitive flag + categories joined with '\n'.
int ref_rules_verdict(void* r, const char* text, size_t len, char* cats, size_t cap) {
  auto v = static_cast<RulesBox*>(r)->set->scan(std::string_view(text, len));
  std::string joined;
  for (size_t i = 0; i < v.categories.size(); ++i) {
    if (i) joined += '\n';
    joined += v.categories[i];
  }
  put_err(cats, cap, joined);
  return v.sensitive ? 1 : 0;
}

// Per-rule hit mask: rule i is tested by a one-rule snapshot built from the same
// PatternRule (the reference scan ORs independent per-rule tests, detection.hpp:153-159,
// except that a later duplicate blacklist term overwrites an earlier one in the
// shared trie, detection.hpp:62 -- reproduced by building the trie-only snapshot
// from ALL blacklist rules and attributing hits by rule index).
void* ref_rules_masker(void* r) {
  auto* box = static_cast<RulesBox*>(r);
  return box;  // masks are computed on the fly in ref_rules_mask
}

// Per-rule hit bits of every rule (bit i of word i / 64 = rule i of the list), any library size.
void ref_rules_mask_wide(void* r, const char* text, size_t len, uint64_t* out, size_t words) {
  const auto& set = *static_cast<RulesBox*>(r)->set;
  const auto& rules = set.rules();
  for (size_t w = 0; w < words; ++w) out[w] = 0;
  auto set_bit = [&](size_t i) {
    if (i / 64 < words) out[i / 64] |= 1ull << (i % 64);
  };
  // regex rules: one snapshot per rule (compiled lazily, cached per call site)
  // cache value keeps the owning snapshot alive so its address cannot be reused
  struct Entry {
    std::shared_ptr<const CompiledRuleSet> owner, compiled;
  };
  static thread_local std::map<std::pair<const void*, size_t>, Entry> cache;
  auto owner = static_cast<RulesBox*>(r)->set;
  for (size_t i = 0; i < rules.size(); ++i) {
    if (rules[i].kind == PatternRule::Kind::ExactBlacklist) continue;
    if (!rules[i].enabled) continue;
    auto key = std::make_pair(static_cast<const void*>(&set), i);
    auto it = cache.find(key);
    if (it == cache.end()) {
      PatternRule one = rules[i];
      it = cache.emplace(key, Entry{owner, CompiledRuleSet::compile({one}, 0)}).first;
    }
    if (it->second.compiled->scan(std::string_view(text, len)).sensitive) set_bit(i);
  }
  // blacklist rules: compile the reference trie with every blacklist rule in order,
  // each tagged by a unique category, so the verdict names the winning rule.
  {
    auto key = std::make_pair(static_cast<const void*>(&set), size_t(1) << 40);
    auto it = cache.find(key);
    if (it == cache.end()) {
      std::vector<PatternRule> only;
      for (size_t i = 0; i < rules.size(); ++i) {
        if (rules[i].kind != PatternRule::Kind::ExactBlacklist) continue;
        PatternRule one = rules[i];
        one.rule_id = "r" + std::to_string(i);
        one.category = std::to_string(i);
        only.push_back(one);
      }
      it = cache.emplace(key, Entry{owner, CompiledRuleSet::compile(only, 0)}).first;
    }
    auto v = it->second.compiled->scan(std::string_view(text, len));
    for (const auto& c : v.categories) set_bit(std::stoul(c));
  }
}

// rules 0..63 (the per-rule masks of the parity tests; wider sets: ref_rules_mask_wide)
uint64_t ref_rules_mask(void* r, const char* text, size_t len) {
  uint64_t m = 0;
  ref_rules_mask_wide(r, text, len, &m, 1);
  return m;
}

// Window verdict masks for every full block of every prompt (Appendix A.3).
// Windows are scanned with a std::thread pool (scans are reentrant on an immutable
// snapshot, detection.hpp:116-117).  out_mask is indexed by the flat block index
// (prompt-major).  Returns the number of blocks.
// stock = 1: ONE CompiledRuleSet::scan per window, exactly as RuleEngine::tier1_scan runs it
// (detection.hpp:148-170, 217); the mask is then 1 for a sensitive window (the label input),
// not the per-rule attribution.  This is the timed reference arm of bench.py.
static uint64_t scan_windows(void* r, const uint32_t* tok, const uint64_t* off, uint32_t n_prompts, uint32_t B,
                             uint32_t W, uint64_t* out_mask, int nthreads, int stock, uint64_t* out_h = nullptr,
                             uint64_t* out_d = nullptr);

uint64_t ref_scan_windows(void* r, const uint32_t* tok, const uint64_t* off, uint32_t n_prompts,
                          uint32_t B, uint32_t W, uint64_t* out_mask, int nthreads) {
  return scan_windows(r, tok, off, n_prompts, B, W, out_mask, nthreads, 0);
}

// With out_h/out_d the same worker threads also compute every block's key (A.2: stages 1-2
// of a prompt run on one pool thread; hashing is reentrant).
static uint64_t scan_windows(void* r, const uint32_t* tok, const uint64_t* off, uint32_t n_prompts, uint32_t B,
                             uint32_t W, uint64_t* out_mask, int nthreads, int stock, uint64_t* out_h,
                             uint64_t* out_d) {
  const CompiledRuleSet& set = *static_cast<RulesBox*>(r)->set;
  std::vector<uint64_t> boff(n_prompts + 1, 0);
  for (uint32_t p = 0; p < n_prompts; ++p) boff[p + 1] = boff[p] + (off[p + 1] - off[p]) / B;
  if (nthreads <= 0) nthreads = static_cast<int>(std::thread::hardware_concurrency());
  std::atomic<uint32_t> next{0};
  auto work = [&] {
    for (;;) {
      uint32_t p = next.fetch_add(1);
      if (p >= n_prompts) break;
      uint64_t L = off[p + 1] - off[p];
      uint64_t n = L / B;
      if (out_h)
        for (uint64_t b = 0, h = 0; b < n; ++b) {
          uint64_t d = block_digest(tok + off[p] + b * B, B);
          h = chain_key(b ? h : 0, d);
          out_h[boff[p] + b] = h;
          out_d[boff[p] + b] = d;
        }
      for (uint64_t b = 0; b < n; ++b) {
        uint64_t s = off[p] + b * B, e = off[p] + std::min<uint64_t>(L, (b + 1) * B + W);
        TokenSeq win(tok + s, tok + e);
        std::string text = detokenize_bytes(win);
        out_mask[boff[p] + b] = stock ? (set.scan(text).sensitive ? 1u : 0u) : ref_rules_mask(r, text.data(), text.size());
      }
    }
  };
  std::vector<std::thread> th;
  for (int i = 0; i < nthreads; ++i) th.emplace_back(work);
  for (auto& t : th) t.join();
  return boff[n_prompts];
}

// ---------------------------------------------------------------- hashing
uint64_t ref_token_seq_digest(const uint32_t* t, size_t n) { return block_digest(t, static_cast<uint32_t>(n)); }

uint64_t ref_fnv1a64_bytes(const uint8_t* p, size_t n) {
  Fnv1a64 f;
  f.update(p, n);
  return f.digest();
}

uint64_t ref_chain(uint64_t prev_h, uint64_t d) { return chain_key(prev_h, d); }

uint64_t ref_block_keys(const uint32_t* tok, const uint64_t* off, uint32_t n_prompts, uint32_t B,
                        uint64_t* out_h, uint64_t* out_d) {
  uint64_t k = 0;
  for (uint32_t p = 0; p < n_prompts; ++p) {
    uint64_t L = off[p + 1] - off[p], n = L / B, h = 0;
    for (uint64_t b = 0; b < n; ++b, ++k) {
      uint64_t d = block_digest(tok + off[p] + b * B, B);
      h = chain_key(b ? h : 0, d);
      out_h[k] = h;
      out_d[k] = d;
    }
  }
  return k;
}

// ---------------------------------------------------------------- engine
struct RefEngine {
  std::shared_ptr<const CompiledRuleSet> rules;
  void* rules_box;
  uint32_t B, W;
  std::unique_ptr<RadixCacheIndex> idx;
  MonitorConfig mcfg;
  std::unique_ptr<EntropyMonitor> mon;
  std::unordered_map<std::string, uint32_t> intern;  // block content (raw token bytes) -> id (exact)
  std::vector<uint64_t> id_digest;                     // id -> token_seq_digest(content)
  struct Pending {
    TokenSeq ids;
    UserId user;
    OwnerClass owner;
    std::vector<uint8_t> labels;  // 0 Private, 1 Public (SensitivityLabel values)
  };
  std::vector<Pending> pending;
  // the last admit's matches, re-expressed in tokens (one KvHandle of B tokens per
  // matched block) for CostModel::ttft and attribute_reuse
  struct Served {
    uint64_t input_tokens = 0;
    UserId user;
    MatchResult m;
  };
  std::vector<Served> served;
  int nthreads = 1;
  int stock_scan = 0;  // 1: one CompiledRuleSet::scan per window (bench reference arm)
  bool pending_labels = false;  // commit leaves new nodes PendingPrivate (insert's label)
  bool budgeted = false;        // A.9: a bounded HBM budget (insert-time make_room)
  std::vector<uint32_t> dropped;  // prompts of the last commit whose insert raised CapacityExhausted
};

void* ref_engine_create(void* rules, uint32_t B, uint32_t W, double jump, uint64_t u_pre_max) {
  auto* e = new RefEngine;
  e->rules_box = rules;
  e->rules = static_cast<RulesBox*>(rules)->set;
  e->B = B;
  e->W = W;
  RadixCacheIndex::Config cfg;
  cfg.budget = TierBudget::from_tokens(1ull << 50, 1ull << 50, 1ull << 50);
  cfg.tiered_demotion = false;
  e->idx = std::make_unique<RadixCacheIndex>(cfg);
  MonitorConfig mc;
  mc.entropy_jump = jump;
  mc.u_pre_max = u_pre_max;
  e->mcfg = mc;
  e->mon = std::make_unique<EntropyMonitor>(*e->idx, mc);
  return e;
}

void ref_engine_free(void* e) { delete static_cast<RefEngine*>(e); }

// RadixCacheIndex::Config::tiered_demotion (before any insert): a fresh index and monitor
// with the same (unbounded) budgets.
int ref_engine_set_tiered(void* ev, int tiered) {
  auto* e = static_cast<RefEngine*>(ev);
  if (!e->pending.empty()) return -1;
  MonitorConfig mc = e->mcfg;
  e->mon.reset();
  RadixCacheIndex::Config cfg;
  cfg.budget = TierBudget::from_tokens(1ull << 50, 1ull << 50, 1ull << 50);
  cfg.tiered_demotion = tiered != 0;
  e->idx = std::make_unique<RadixCacheIndex>(cfg);
  e->mon = std::make_unique<EntropyMonitor>(*e->idx, mc);
  return 0;
}

// A.9 (bounded budgets): RadixCacheIndex::Config::budget = TierBudget::from_tokens(hbm, dram, ssd)
// in blocks (one interned token per block), before any insert.  The commit then runs the
// serving contract of ServingSimulator::submit (serving_sim.hpp:195-215) for the batch: every
// prompt's matched path stays pinned from its lookup until the batch's inserts are done, each
// insert makes room for its new blocks (cache_index.hpp:183-190, 801-806: evicting unpinned
// leaves), and an insert that cannot make room raises CapacityExhausted -- that prompt is dropped
// (nothing inserted) and the next one is inserted.
int ref_engine_set_budget(void* ev, uint64_t hbm, uint64_t dram, uint64_t ssd, int tiered) {
  auto* e = static_cast<RefEngine*>(ev);
  if (!e->pending.empty()) return -1;
  MonitorConfig mc = e->mcfg;
  e->mon.reset();
  RadixCacheIndex::Config cfg;
  cfg.budget = TierBudget::from_tokens(hbm, dram, ssd);
  cfg.tiered_demotion = tiered != 0;
  e->idx = std::make_unique<RadixCacheIndex>(cfg);
  e->mon = std::make_unique<EntropyMonitor>(*e->idx, mc);
  e->budgeted = true;
  return 0;
}

// prompts dropped by the last commit (A.9), ascending
size_t ref_engine_dropped(void* ev, uint32_t* out, size_t cap) {
  auto* e = static_cast<RefEngine*>(ev);
  for (size_t i = 0; i < e->dropped.size() && i < cap; ++i) out[i] = e->dropped[i];
  return e->dropped.size();
}

// the index's used tokens (= blocks) per tier
void ref_engine_budget_used(void* ev, uint64_t* used3) {
  auto* e = static_cast<RefEngine*>(ev);
  for (int t = 0; t < 3; ++t) used3[t] = e->idx->budget().used(static_cast<MemTier>(t));
}

void ref_engine_set_threads(void* e, int n) { static_cast<RefEngine*>(e)->nthreads = n; }

// Hot reload between batches: the next admit scans with the new snapshot (RuleEngine::load_rules
// swaps the active set atomically, detection.hpp:238-241; in-flight scans keep the old one -- in
// the batched contract a batch is one scan, so the swap lands at a batch boundary).
void ref_engine_set_rules(void* ev, void* rules) {
  auto* e = static_cast<RefEngine*>(ev);
  e->rules_box = rules;
  e->rules = static_cast<RulesBox*>(rules)->set;
}
void ref_engine_set_stock_scan(void* e, int on) { static_cast<RefEngine*>(e)->stock_scan = on; }

// Phase L of Appendix A.1 for one batch: hashes, window verdicts, labels, lookups and
// monitor records (in prompt order).  Per-block outputs are prompt-major flat arrays.
// decision: 0 = not matched, 1 = public hit, 2 = owner hit (private visible to creator).
int ref_engine_admit(void* ev, const uint32_t* tok, const uint64_t* off, const uint64_t* users,
                     const uint8_t* owners, uint32_t n_prompts, uint64_t* out_h, uint64_t* out_d,
                     uint64_t* out_mask, uint8_t* out_label, uint8_t* out_decision,
                     uint32_t* out_matched, uint8_t* out_tier) {
  auto* e = static_cast<RefEngine*>(ev);
  const uint32_t B = e->B;
  std::vector<uint64_t> boff(n_prompts + 1, 0);
  for (uint32_t p = 0; p < n_prompts; ++p) boff[p + 1] = boff[p] + (off[p + 1] - off[p]) / B;
  uint64_t nblk = boff[n_prompts];
  std::vector<uint64_t> mask(nblk);
  scan_windows(e->rules_box, tok, off, n_prompts, B, e->W, mask.data(), e->nthreads, e->stock_scan, out_h, out_d);
  e->pending.clear();
  e->served.assign(n_prompts, {});
  for (uint32_t p = 0; p < n_prompts; ++p) {
    uint64_t n = boff[p + 1] - boff[p];
    RefEngine::Pending pd;
    pd.user = UserId{users[p]};
    pd.owner = owners[p] ? OwnerClass::Business : OwnerClass::Customer;
    bool priv = false;
    for (uint64_t b = 0; b < n; ++b) {
      uint64_t k = boff[p] + b;
      out_mask[k] = mask[k];
      priv = priv || mask[k] != 0;  // A.4 inherited sensitivity (prefix-OR)
      uint8_t lbl = priv ? static_cast<uint8_t>(SensitivityLabel::Private)
                         : static_cast<uint8_t>(SensitivityLabel::Public);
      out_label[k] = lbl;
      pd.labels.push_back(lbl);
      std::string content = content_key(tok + off[p] + b * B, B);
      auto it = e->intern.find(content);
      uint32_t id;
      if (it == e->intern.end()) {
        id = static_cast<uint32_t>(e->id_digest.size());
        e->intern.emplace(content, id);
        e->id_digest.push_back(out_d[k]);
      } else {
        id = it->second;
      }
      pd.ids.push_back(id);
    }
    uint32_t m = 0;
    uint8_t tier = 0;
    if (n > 0) {
      MatchResult mr = e->idx->match_prefix(pd.ids, pd.user);
      m = static_cast<uint32_t>(mr.matched_tokens);
      tier = static_cast<uint8_t>(mr.lowest_tier);
      for (size_t b = 0; b < mr.path.size(); ++b) {
        NodeRef nd = mr.path[b];
        out_decision[boff[p] + b] = nd->label == SensitivityLabel::Public ? 1 : 2;
        e->mon->record_access(nd, pd.user);
      }
      RefEngine::Served& sv = e->served[p];
      sv.m = mr;
      sv.m.matched_tokens = mr.matched_tokens * B;
      for (KvHandle& h : sv.m.handles) h.token_count = B;
    }
    e->served[p].input_tokens = off[p + 1] - off[p];
    e->served[p].user = pd.user;
    for (uint64_t b = m; b < n; ++b) out_decision[boff[p] + b] = 0;
    out_matched[p] = m;
    out_tier[p] = tier;
    e->pending.push_back(std::move(pd));
  }
  return 0;
}

// Serving observables of the last admit: CostModel::ttft (serving_sim.hpp:50-56) on the
// token-scaled match, and ServingSimulator::attribute_reuse (serving_sim.hpp:313-324,
// private there, restated here line for line with node span = B tokens).
int ref_engine_ttft(void* ev, const uint64_t* request_ids, double t_base, double c_prefill, double pen_dram,
                    double pen_ssd, double sigma, uint64_t seed, double* out_ttft, uint32_t* out_intra,
                    uint32_t* out_inter) {
  auto* e = static_cast<RefEngine*>(ev);
  CostModel cm;
  cm.t_base_ms = t_base;
  cm.c_prefill_ms = c_prefill;
  cm.tier_penalty_ms = {0.0, pen_dram, pen_ssd};
  cm.noise_sigma_ms = sigma;
  cm.seed = seed;
  for (size_t p = 0; p < e->served.size(); ++p) {
    const auto& sv = e->served[p];
    out_ttft[p] = cm.ttft(sv.input_tokens, sv.m, request_ids ? request_ids[p] : p);
    uint64_t counted = 0, intra = 0, inter = 0;
    for (size_t i = 0; i < sv.m.path.size(); ++i) {
      NodeRef n = sv.m.path[i];
      uint64_t covered = std::min<uint64_t>(static_cast<uint64_t>(n->span()) * e->B, sv.m.matched_tokens - counted);
      counted += covered;
      if (n->creator == sv.user)
        intra += covered;
      else
        inter += covered;
    }
    out_intra[p] = static_cast<uint32_t>(intra);
    out_inter[p] = static_cast<uint32_t>(inter);
  }
  return 0;
}

void ref_engine_set_pending(void* ev, int pending) { static_cast<RefEngine*>(ev)->pending_labels = pending != 0; }

// Label landing: RadixCacheIndex::resolve_block (cache_index.hpp:321-343) of each prompt's
// span [first[p], n_p) with labels[p] (propagate = the label is private), in the batched
// order of skv_resolve_blocks: all Public landings, then Private, then Restricted.
int ref_engine_resolve(void* ev, const uint32_t* tok, const uint64_t* off, uint32_t n_prompts, const uint32_t* first,
                       const uint8_t* labels) {
  auto* e = static_cast<RefEngine*>(ev);
  const uint32_t B = e->B;
  const uint8_t order[3] = {static_cast<uint8_t>(SensitivityLabel::Public),
                            static_cast<uint8_t>(SensitivityLabel::Private),
                            static_cast<uint8_t>(SensitivityLabel::Restricted)};
  for (uint8_t want : order) {
    for (uint32_t p = 0; p < n_prompts; ++p) {
      if (labels[p] != want) continue;
      const uint64_t n = (off[p + 1] - off[p]) / B;
      if (first[p] >= n) continue;
      TokenSeq ids;
      for (uint64_t b = 0; b < n; ++b) {
        std::string content = content_key(tok + off[p] + b * B, B);
        auto it = e->intern.find(content);
        if (it == e->intern.end()) return -1;
        ids.push_back(it->second);
      }
      NodeRef terminal = e->idx->find_node(ids);
      if (!terminal) return -1;
      const auto lab = static_cast<SensitivityLabel>(want);
      const bool priv = lab != SensitivityLabel::Public;
      e->idx->resolve_block(terminal, static_cast<uint32_t>(n - first[p]), lab, priv, priv ? 0 : 1);
    }
  }
  return 0;
}

// Phase C (A.7): insert in prompt order, one node per block, labels applied per block.
int ref_engine_commit(void* ev) {
  auto* e = static_cast<RefEngine*>(ev);
  e->dropped.clear();
  // A.9: the batch's matched paths stay pinned through its inserts (serving_sim.hpp:196,215)
  std::vector<NodeRef> pins;
  if (e->budgeted)
    for (auto& sv : e->served)
      for (NodeRef n : sv.m.path) {
        e->idx->pin(n);
        pins.push_back(n);
      }
  uint32_t pi = 0;
  for (auto& pd : e->pending) {
    const uint32_t p = pi++;
    size_t n = pd.ids.size();
    if (n == 0) continue;
    uint32_t fresh = 0;
    if (e->budgeted) {
      try {
        e->idx->insert(pd.ids, pd.user, pd.owner, e->idx->current_epoch(), &fresh);
      } catch (const CapacityExhausted&) {
        e->dropped.push_back(p);
        continue;
      }
    } else {
      e->idx->insert(pd.ids, pd.user, pd.owner, e->idx->current_epoch(), &fresh);
    }
    if (fresh == 0) continue;
    size_t k0 = n - fresh;
    for (size_t k = k0 + 1; k < n; ++k) e->idx->ensure_boundary(pd.ids, k);
    if (e->pending_labels) continue;
    for (size_t b = k0; b < n; ++b) {
      TokenSeq pre(pd.ids.begin(), pd.ids.begin() + b + 1);
      NodeRef nd = e->idx->find_node(pre);
      if (!nd) return -1;
      if (pd.labels[b] == static_cast<uint8_t>(SensitivityLabel::Public))
        e->idx->set_label(nd, SensitivityLabel::Public, false, 1);
      else
        e->idx->set_label(nd, SensitivityLabel::Private, true);
    }
  }
  for (NodeRef n : pins) e->idx->unpin(n);
  e->pending.clear();
  return 0;
}

// Set tier tags on existing entries: tiers[k] (0 HBM, 1 DRAM, 2 SSD) for every full
// block of every prompt, applied with RadixCacheIndex::demote (cache_index.hpp:362-381).
// RadixCacheIndex::evict(needed, epoch) (cache_index.hpp:281-292) on the reference index;
// *n_out = nodes freed.  Returns 1 when the reference ran out of candidates
// (CapacityExhausted) after freeing what it could.
int ref_engine_evict(void* ev, uint64_t needed, uint64_t epoch, uint64_t* n_out) {
  auto* e = static_cast<RefEngine*>(ev);
  // nodes holding HBM handles: freeing or demoting a victim removes one
  auto count = [&] {
    uint64_t n = 0;
    e->idx->for_each_node([&](const CacheNode* nd) {
      for (const KvHandle& h : nd->kv_handles)
        if (h.tier == MemTier::HBM) {
          ++n;
          break;
        }
    });
    return n;
  };
  const uint64_t before = count();
  int rc = 0;
  try {
    e->idx->evict(needed, epoch);
  } catch (const CapacityExhausted&) {
    rc = 1;
  }
  *n_out = before - count();
  return rc;
}

uint64_t ref_engine_current_epoch(void* ev) { return static_cast<RefEngine*>(ev)->idx->current_epoch(); }

int ref_engine_set_tiers(void* ev, const uint32_t* tok, const uint64_t* off, uint32_t n_prompts,
                         const uint8_t* tiers) {
  auto* e = static_cast<RefEngine*>(ev);
  uint64_t k = 0;
  for (uint32_t p = 0; p < n_prompts; ++p) {
    uint64_t n = (off[p + 1] - off[p]) / e->B;
    TokenSeq ids;
    for (uint64_t b = 0; b < n; ++b, ++k) {
      std::string content = content_key(tok + off[p] + b * e->B, e->B);
      auto it = e->intern.find(content);
      if (it == e->intern.end()) return -1;
      ids.push_back(it->second);
      NodeRef nd = e->idx->find_node(ids);
      if (!nd || nd->kv_handles.empty()) return -2;
      while (static_cast<uint8_t>(nd->kv_handles[0].tier) < tiers[k]) e->idx->demote(nd->kv_handles[0]);
    }
  }
  return 0;
}

// One monitor epoch (A.6).  Events are written in reference visit order; keys are the
// (h, d) of the event node's block path.
int ref_engine_epoch(void* ev, uint64_t* out_epoch, size_t cap, uint64_t* ev_h, uint64_t* ev_d,
                     uint8_t* ev_action, double* ev_now, double* ev_prev, uint64_t* ev_upre,
                     size_t* n_events) {
  auto* e = static_cast<RefEngine*>(ev);
  uint64_t epoch = e->idx->advance_epoch();
  auto fired = e->mon->epoch_pass(epoch);
  *out_epoch = epoch;
  // node -> key by walking parents
  auto key_of = [&](const CacheNode* nd, uint64_t* h, uint64_t* d) {
    std::vector<const CacheNode*> chain;
    for (const CacheNode* c = nd; !c->is_root(); c = c->parent) chain.push_back(c);
    uint64_t hh = 0, dd = 0;
    for (auto it = chain.rbegin(); it != chain.rend(); ++it) {
      dd = e->id_digest[(*it)->edge[0]];
      hh = chain_key(it == chain.rbegin() ? 0 : hh, dd);
    }
    *h = hh;
    *d = dd;
  };
  size_t i = 0;
  for (const auto& a : fired) {
    if (i < cap) {
      key_of(a.node, &ev_h[i], &ev_d[i]);
      ev_action[i] = static_cast<uint8_t>(a.action);
      ev_now[i] = a.entropy_now;
      ev_prev[i] = a.entropy_prev;
      ev_upre[i] = a.u_pre;
    }
    ++i;
  }
  *n_events = i;
  return 0;
}

// Export every node: key, creator, label, owner, tier, window stats.  Returns count.
size_t ref_engine_export(void* ev, size_t cap, uint64_t* h, uint64_t* d, uint64_t* creator,
                         uint8_t* label, uint8_t* owner, uint8_t* tier, uint64_t* hit_cur,
                         uint64_t* u_cnt, uint64_t* hit_pre, uint64_t* u_pre) {
  auto* e = static_cast<RefEngine*>(ev);
  size_t i = 0;
  std::unordered_map<const CacheNode*, uint64_t> hmap;
  e->idx->for_each_node([&](const CacheNode* nd) {
    uint64_t dd = e->id_digest[nd->edge[0]];
    uint64_t ph = nd->parent->is_root() ? 0 : hmap.at(nd->parent);
    uint64_t hh = chain_key(ph, dd);
    hmap[nd] = hh;
    if (i < cap) {
      h[i] = hh;
      d[i] = dd;
      creator[i] = nd->creator.value;
      label[i] = static_cast<uint8_t>(nd->label);
      owner[i] = static_cast<uint8_t>(nd->owner_class);
      tier[i] = nd->kv_handles.empty() ? 0 : static_cast<uint8_t>(nd->kv_handles[0].tier);
      hit_cur[i] = nd->stats.hit_cur;
      u_cnt[i] = nd->stats.u_cnt;
      hit_pre[i] = nd->stats.hit_pre;
      u_pre[i] = nd->stats.u_pre;
    }
    ++i;
  });
  return i;
}

// ---------------------------------------------------------------- workload
struct WlBox {
  Workload wl;
};

void* ref_workload_generate(int scenario, uint64_t n_users, uint64_t n_requests, double inter,
                            double intra, double secret_density, double ctx_frac, uint64_t seed,
                            char* err, size_t errcap) {
  try {
    WorkloadSpec s;
    s.scenario = static_cast<ScenarioKind>(scenario);
    s.n_users = n_users;
    s.n_requests = n_requests;
    s.inter_user_overlap = inter;
    s.intra_user_overlap = intra;
    s.secret_density = secret_density;
    s.context_dependent_fraction = ctx_frac;
    s.seed = seed;
    return new WlBox{generate(s)};
  } catch (const std::exception& e) {
    put_err(err, errcap, e.what());
    return nullptr;
  }
}

void ref_workload_free(void* w) { delete static_cast<WlBox*>(w); }
size_t ref_workload_count(void* w) { return static_cast<WlBox*>(w)->wl.requests.size(); }
uint64_t ref_workload_digest(void* w) { return fnv1a64(static_cast<WlBox*>(w)->wl.canonical_bytes()); }
size_t ref_workload_text(void* w, size_t i, char* out, size_t cap) {
  const auto& t = static_cast<WlBox*>(w)->wl.requests[i].text;
  if (out && cap >= t.size()) std::memcpy(out, t.data(), t.size());
  return t.size();
}
uint64_t ref_workload_user(void* w, size_t i) { return static_cast<WlBox*>(w)->wl.requests[i].user.value; }
uint8_t ref_workload_owner(void* w, size_t i) {
  return static_cast<uint8_t>(static_cast<WlBox*>(w)->wl.requests[i].owner);
}
// Ground truth spans: begin/end/sensitivity(0 Always, 1 ContextOnly).
size_t ref_workload_truth(void* w, size_t i, size_t cap, uint64_t* begin, uint64_t* end, uint8_t* sens) {
  const auto& tr = static_cast<WlBox*>(w)->wl.requests[i].truth;
  for (size_t k = 0; k < tr.size() && k < cap; ++k) {
    begin[k] = tr[k].begin;
    end[k] = tr[k].end;
    sens[k] = static_cast<uint8_t>(tr[k].sensitivity);
  }
  return tr.size();
}

// safekv::block_truth (workload.hpp:137-147) of request i's byte range [begin, end).
void ref_workload_block_truth(void* w, size_t i, size_t begin, size_t end, int* alone, int* with_ctx) {
  BlockTruth t = block_truth(static_cast<WlBox*>(w)->wl.requests[i], begin, end);
  *alone = t.sensitive_alone ? 1 : 0;
  *with_ctx = t.sensitive_with_context ? 1 : 0;
}

// Generator primitives (workload.hpp:155-266), exposed so tests can pin the
// product-side synthetic generator against the reference byte for byte.
size_t ref_filler(uint64_t uniq, size_t n, uint64_t* rng_state, char* out) {
  // SplitMix64 has no state accessor; replay by constructing from a seed and
  // advancing is not possible, so the harness keeps its own SplitMix64 per call:
  // *rng_state is the seed on input and is unused on output.
  SplitMix64 rng(*rng_state);
  std::string s = detail::filler(uniq, n, rng);
  std::memcpy(out, s.data(), s.size());
  return s.size();
}

size_t ref_make_secret(size_t family, uint64_t seed, char* out, size_t cap) {
  SplitMix64 rng(seed);
  auto s = detail::make_secret(family, rng);
  if (cap >= s.text.size()) std::memcpy(out, s.text.data(), s.text.size());
  return s.text.size();
}

uint64_t ref_derive_seed(uint64_t root, uint64_t tag) { return derive_seed(root, tag); }

size_t ref_rule_corpus(size_t n, uint64_t seed, char* out, size_t cap, uint32_t* lens) {
  auto c = generate_rule_corpus(n, seed);
  size_t pos = 0;
  for (size_t i = 0; i < c.size(); ++i) {
    lens[i] = static_cast<uint32_t>(c[i].first.size());
    if (pos + c[i].first.size() <= cap) std::memcpy(out + pos, c[i].first.data(), c[i].first.size());
    pos += c[i].first.size();
  }
  return pos;
}

}  // extern "C"
