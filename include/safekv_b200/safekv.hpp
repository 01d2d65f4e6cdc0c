// safekv.hpp -- header-only C++ facade over the C ABI (include/safekv_b200.h) that keeps the
// reference's class and method names for the admission path (reference
// proj/include/safekv/{core,detection,cache_index,monitor}.hpp), so a caller such as
// ServingSimulator::submit (serving_sim.hpp:184-218) can switch to the device path with a
// type swap.  Every call goes to the CUDA library; errors are rethrown as
// the reference's exception classes (core.hpp:19-59).
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "../safekv_b200.h"

namespace safekv_b200 {

// ---- errors (core.hpp:19-59) -------------------------------------------------------
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CapacityExhausted : Error {
  using Error::Error;
};
struct ParseError : Error {
  using Error::Error;
};
struct CompileError : Error {
  using Error::Error;
};
struct ConfigError : Error {
  using Error::Error;
};
struct DeviceError : Error {
  using Error::Error;
};

inline void check(int rc, const std::string& msg) {
  switch (rc) {
    case SKV_OK: return;
    case SKV_ERR_PARSE: throw ParseError(msg);
    case SKV_ERR_COMPILE: throw CompileError(msg);
    case SKV_ERR_CONFIG: throw ConfigError(msg);
    case SKV_ERR_CAPACITY: throw CapacityExhausted(msg);
    case SKV_ERR_CUDA: throw DeviceError(msg);
    default: throw Error(msg);
  }
}

// ---- vocabulary (core.hpp:65-176) ---------------------------------------------------
using TokenId = uint32_t;
using TokenSeq = std::vector<TokenId>;
struct UserId {
  uint64_t value = 0;
};
enum class OwnerClass : uint8_t { Customer = 0, Business = 1 };
enum class MemTier : uint8_t { HBM = 0, DRAM = 1, SSD = 2 };
enum class SensitivityLabel : uint8_t { Private = 0, Public = 1, PendingPrivate = 2, Restricted = 3 };
enum class AnomalyAction : uint8_t { None = 0, DowngradeToPrivate = 1, Restrict = 2 };

// detection.hpp:36-42
struct DetectionVerdict {
  bool sensitive = false;
  int tier = 1;
  double score = 0.0;
  std::vector<std::string> categories;
  bool escalate = false;
};

// monitor.hpp:21-30 (entries are identified by their key instead of a CacheNode*)
struct AnomalyEvent {
  uint64_t key_h = 0, key_d = 0;
  double entropy_now = 0.0, entropy_prev = 0.0;
  uint64_t u_pre = 0;
  AnomalyAction action = AnomalyAction::None;
  uint64_t epoch = 0;
  OwnerClass owner_class = OwnerClass::Customer;
};

// ---- CompiledRuleSet (detection.hpp:118-181): immutable compiled snapshot ----------
class CompiledRuleSet {
 public:
  static std::shared_ptr<const CompiledRuleSet> defaults() {
    skv_rules* r = nullptr;
    check(skv_rules_default(&r), "default rules");
    return std::shared_ptr<const CompiledRuleSet>(new CompiledRuleSet(r));
  }
  // RuleEngine::load_rules_json (detection.hpp:222-242)
  static std::shared_ptr<const CompiledRuleSet> from_json(const std::string& json,
                                                          std::vector<std::string>* warnings = nullptr) {
    skv_rules* r = nullptr;
    char err[1024] = {0};
    const int rc = skv_rules_from_json(json.data(), json.size(), &r, err, sizeof(err));
    check(rc, err);
    auto set = std::shared_ptr<const CompiledRuleSet>(new CompiledRuleSet(r));
    if (warnings)
      for (size_t i = 0; i < skv_rules_warning_count(r); ++i) warnings->emplace_back(skv_rules_warning(r, i));
    return set;
  }
  ~CompiledRuleSet() { skv_rules_free(r_); }
  CompiledRuleSet(const CompiledRuleSet&) = delete;
  CompiledRuleSet& operator=(const CompiledRuleSet&) = delete;

  size_t size() const { return skv_rules_count(r_); }
  uint64_t version() const { return skv_rules_version(r_); }
  const skv_rules* handle() const { return r_; }

  // u32 words of a window's device mask (more than 32 enabled rules: several)
  uint32_t mask_words() const { return skv_rules_mask_words(r_); }

  // verdict of a device rule mask, in the reference's category order (detection.hpp:160-169)
  DetectionVerdict verdict(uint32_t device_mask) const { return verdict(&device_mask, 1); }
  // ... of a mask of mask_words() words, word w at words[w * stride]
  DetectionVerdict verdict(const uint32_t* words, size_t stride) const {
    DetectionVerdict v;
    std::vector<bool> hit(size(), false);
    for (uint32_t j = 0; j < skv_rules_enabled_count(r_); ++j)
      if (words[(j / 32) * stride] >> (j % 32) & 1u) hit[skv_rules_enabled_rule(r_, j)] = true;
    for (uint32_t i = 0; i < size(); ++i) {
      if (!hit[i]) continue;
      const char* cat = nullptr;
      skv_rules_info(r_, i, nullptr, &cat, nullptr, nullptr);
      v.sensitive = true;
      bool seen = false;
      for (const auto& c : v.categories) seen = seen || c == cat;
      if (!seen) v.categories.emplace_back(cat);
    }
    v.score = v.sensitive ? 1.0 : 0.0;
    v.escalate = !v.sensitive;
    return v;
  }

 private:
  explicit CompiledRuleSet(skv_rules* r) : r_(r) {}
  skv_rules* r_;
};

// ---- AdmissionIndex: device-resident RadixCacheIndex + EntropyMonitor + rule tier -----
class AdmissionIndex {
 public:
  struct Request {
    const TokenSeq* tokens;
    UserId user;
    OwnerClass owner = OwnerClass::Customer;
  };
  // per-batch outputs (phase L)
  struct Admission {
    std::vector<uint64_t> block_offsets;  // n + 1
    std::vector<uint64_t> key_h, key_d;   // per block
    std::vector<uint8_t> labels;          // SensitivityLabel per block
    std::vector<uint32_t> rule_masks;     // device rule mask per block (word 0; skv_last_rule_masks: all)
    std::vector<uint8_t> decisions;       // 0 miss, 1 public hit, 2 owner hit
    std::vector<uint32_t> matched_blocks; // per request
    std::vector<MemTier> lowest_tier;     // per request
  };
  // MatchResult subset that survives the flat representation (cache_index.hpp:100-106)
  struct MatchResult {
    uint64_t matched_tokens = 0;
    MemTier lowest_tier = MemTier::HBM;
  };

  explicit AdmissionIndex(const skv_config* cfg = nullptr) {
    skv_config c;
    skv_config_default(&c);
    if (cfg) c = *cfg;
    block_tokens_ = c.block_tokens;
    skv_ctx* ctx = nullptr;
    int rc = skv_create(&c, &ctx);
    check(rc, skv_last_error(nullptr));
    ctx_ = ctx;
    rules_ = CompiledRuleSet::defaults();
  }
  ~AdmissionIndex() { skv_destroy(ctx_); }

  // the status is computed before the error string is fetched (argument order is unspecified)
  void ok(int rc) const { check(rc, skv_last_error(ctx_)); }
  AdmissionIndex(const AdmissionIndex&) = delete;
  AdmissionIndex& operator=(const AdmissionIndex&) = delete;

  // RuleEngine::load_rules_json + atomic snapshot swap (detection.hpp:222-242)
  std::shared_ptr<const CompiledRuleSet> load_rules_json(const std::string& json,
                                                         std::vector<std::string>* warnings = nullptr) {
    auto set = CompiledRuleSet::from_json(json, warnings);
    ok(skv_set_rules(ctx_, set->handle()));
    rules_ = set;
    return set;
  }
  std::shared_ptr<const CompiledRuleSet> active() const { return rules_; }

  // RuleEngine::tier1_scan (detection.hpp:217)
  DetectionVerdict tier1_scan(std::string_view text) {
    std::vector<uint32_t> mask(std::max<uint32_t>(1, skv_mask_words(ctx_)), 0);
    ok(skv_tier1_scan(ctx_, text.data(), text.size(), mask.data()));
    return rules_->verdict(mask.data(), 1);
  }

  // token_seq_digest (core.hpp:68-73)
  uint64_t token_seq_digest(const TokenSeq& seq) {
    uint64_t d = 0;
    ok(skv_token_seq_digest(ctx_, seq.data(), seq.size(), &d));
    return d;
  }

  // Phase L for a batch: hash, scan, label, lookup, record accesses.
  Admission admit(const std::vector<Request>& reqs) {
    std::vector<uint32_t> toks;
    std::vector<uint64_t> off{0}, users;
    std::vector<uint8_t> owners;
    for (const auto& r : reqs) {
      toks.insert(toks.end(), r.tokens->begin(), r.tokens->end());
      off.push_back(toks.size());
      users.push_back(r.user.value);
      owners.push_back(static_cast<uint8_t>(r.owner));
    }
    const uint32_t n = static_cast<uint32_t>(reqs.size());
    uint64_t nb = 0;
    for (uint32_t p = 0; p < n; ++p) nb += (off[p + 1] - off[p]) / block_tokens_;
    Admission a;
    a.block_offsets.resize(n + 1);
    a.key_h.resize(nb);
    a.key_d.resize(nb);
    a.labels.resize(nb);
    a.rule_masks.resize(nb);
    a.decisions.resize(nb);
    a.matched_blocks.resize(n);
    std::vector<uint8_t> tiers(n);
    std::vector<uint32_t> boff(n + 1);
    skv_batch b{toks.data(), off.data(), users.data(), owners.data(), n, toks.size(), 0};
    skv_admit_out o{a.key_h.data(), a.key_d.data(), a.labels.data(), a.rule_masks.data(), a.decisions.data(),
                    a.matched_blocks.data(), tiers.data(), nullptr, 0, 0, 0};
    ok(skv_admit(ctx_, &b, &o));
    for (uint32_t p = 0, acc = 0; p <= n; ++p) {
      a.block_offsets[p] = acc;
      if (p < n) acc += static_cast<uint32_t>((off[p + 1] - off[p]) / block_tokens_);
    }
    a.lowest_tier.reserve(n);
    for (uint8_t t : tiers) a.lowest_tier.push_back(static_cast<MemTier>(t));
    return a;
  }

  // Phase C: insert the last admitted batch (first creator wins).  Returns new entries.
  uint64_t commit() {
    uint64_t nn = 0;
    ok(skv_commit(ctx_, &nn));
    return nn;
  }

  // Phase E: advance_epoch + EntropyMonitor::epoch_pass (monitor.hpp:85-99)
  std::vector<AnomalyEvent> epoch_pass() {
    std::vector<skv_event> buf(1 << 16);
    size_t n = 0;
    uint64_t ep = 0;
    ok(skv_epoch(ctx_, buf.data(), buf.size(), &n, &ep));
    if (n > buf.size()) throw CapacityExhausted("more anomaly events than the facade buffer");
    std::vector<AnomalyEvent> out;
    for (size_t i = 0; i < n; ++i) {
      const skv_event& e = buf[i];
      out.push_back(AnomalyEvent{e.h, e.d, e.entropy_now, e.entropy_prev, e.u_pre,
                                 static_cast<AnomalyAction>(e.action), e.epoch, static_cast<OwnerClass>(e.owner)});
    }
    return out;
  }

  // RadixCacheIndex::match_prefix (cache_index.hpp:213-237) as a batch of one, block
  // granular (A.5).  Like the reference call it records nothing permanent in the index:
  // the batch is admitted (its accesses counted, as submit() does right after) but not
  // committed.
  MatchResult match_prefix(const TokenSeq& seq, UserId user) {
    Admission a = admit({Request{&seq, user}});
    return MatchResult{static_cast<uint64_t>(a.matched_blocks[0]) * block_tokens_, a.lowest_tier[0]};
  }

  // RadixCacheIndex::insert of one sequence (admit + commit of a batch of one).
  uint64_t insert(const TokenSeq& seq, UserId user, OwnerClass owner) {
    admit({Request{&seq, user, owner}});
    return commit();
  }

  // CostModel (serving_sim.hpp:25-57); CostModel::validate failures throw ConfigError
  struct CostModel {
    double t_base_ms = 10.0;
    double c_prefill_ms = 1.0;
    double tier_penalty_ms[3] = {0.0, 0.2, 0.5};  // HBM, DRAM, SSD
    double noise_sigma_ms = 0.0;
    uint64_t seed = 0;
  };
  void set_cost_model(const CostModel& m) {
    skv_cost_model c{m.t_base_ms, m.c_prefill_ms, {m.tier_penalty_ms[0], m.tier_penalty_ms[1], m.tier_penalty_ms[2]},
                     m.noise_sigma_ms, m.seed};
    ok(skv_set_cost_model(ctx_, &c));
  }
  // Per request of the last admit: CostModel::ttft (serving_sim.hpp:50-56) and the
  // reuse attribution of ServingSimulator::attribute_reuse (serving_sim.hpp:313-324).
  struct Served {
    std::vector<double> ttft_ms;
    std::vector<uint32_t> intra_tokens, inter_tokens;
  };
  Served served(size_t n_requests, const std::vector<uint64_t>* request_ids = nullptr) {
    Served s;
    s.ttft_ms.resize(n_requests);
    s.intra_tokens.resize(n_requests);
    s.inter_tokens.resize(n_requests);
    ok(skv_admit_ttft(ctx_, request_ids ? request_ids->data() : nullptr, s.ttft_ms.data(), s.intra_tokens.data(),
                      s.inter_tokens.data(), 0));
    return s;
  }

  // RadixCacheIndex::evict (cache_index.hpp:281-292).  enable_eviction() must precede
  // the first admit (RadixCacheIndex::Config::tiered_demotion selects demotion to DRAM
  // instead of freeing).  Returns the victims' keys (h, d); throws CapacityExhausted, like
  // the reference, when fewer than needed blocks could be freed.
  void enable_eviction(bool tiered_demotion = false) { ok(skv_enable_eviction(ctx_, tiered_demotion ? 1 : 0)); }
  std::vector<std::pair<uint64_t, uint64_t>> evict(uint64_t needed_blocks, uint64_t epoch = 0) {
    std::vector<uint64_t> h(needed_blocks), d(needed_blocks);
    uint64_t n = 0;
    const int rc = skv_evict(ctx_, needed_blocks, epoch, &n, h.data(), d.data(), h.size());
    std::vector<std::pair<uint64_t, uint64_t>> out;
    for (uint64_t i = 0; i < n && i < h.size(); ++i) out.emplace_back(h[i], d[i]);
    ok(rc);
    return out;
  }

  uint64_t entry_count() { return skv_entry_count(ctx_); }
  skv_ctx* handle() { return ctx_; }

 private:
  skv_ctx* ctx_ = nullptr;
  uint32_t block_tokens_ = 16;
  std::shared_ptr<const CompiledRuleSet> rules_;
};

}  // namespace safekv_b200
