// detection.hpp -- drop-in facade of the reference's detection header (proj/include/safekv/
// detection.hpp:28-677): PatternRule, DetectionVerdict, CompiledRuleSet (an immutable compiled
// snapshot), the hot-reloadable RuleEngine, the Tier-2/3 detector mocks, adaptive thresholding and
// the asynchronous DetectionPipeline with its index sink.  Rule sets compile on the host into the
// search DFA the device scans (skv_rules_*); scan() runs on the device (skv_tier1_scan) against the
// snapshot it is called on, and a pipeline drain runs the Tier-1 scan of every drained block in one
// launch (skv_tier1_scan_batch).  Tier-2/3 are the reference's seeded mocks (or an attached
// ExternalDetectorClient): stand-ins for out-of-process detectors, evaluated in drain order on the
// host exactly as the reference does, so their seeded streams stay bit-reproducible.  Their labels
// land in the device index through make_index_sink -> RadixCacheIndex::resolve_block.
#pragma once

#include <cmath>
#include <deque>
#include <fstream>
#include <functional>
#include <memory>
#include <optional>
#include <mutex>
#include <nlohmann/json.hpp>
#include <sstream>
#include <string>
#include <string_view>
#include <vector>

#include "cache_index.hpp"
#include "core.hpp"

namespace safekv {

struct PatternRule {
  std::string rule_id;
  std::string category;
  enum class Kind : uint8_t { Regex, ExactBlacklist } kind = Kind::Regex;
  std::string pattern;
  bool enabled = true;
};

struct DetectionVerdict {
  bool sensitive = false;
  int tier = 1;
  double score = 0.0;
  std::vector<std::string> categories;
  bool escalate = false;
};

class CompiledRuleSet {
 public:
  // detection.hpp:120-144 (CompileError names the rule; duplicate rule_id rejected)
  static std::shared_ptr<const CompiledRuleSet> compile(std::vector<PatternRule> rules, uint64_t version) {
    nlohmann::json j;
    j["version"] = version;
    j["rules"] = nlohmann::json::array();
    for (const auto& r : rules)
      j["rules"].push_back({{"rule_id", r.rule_id},
                            {"category", r.category},
                            {"kind", r.kind == PatternRule::Kind::Regex ? "regex" : "blacklist"},
                            {"pattern", r.pattern},
                            {"enabled", r.enabled}});
    return from_json_text(j.dump(), nullptr);
  }

  static std::shared_ptr<const CompiledRuleSet> from_json_text(const std::string& text,
                                                               std::vector<std::string>* warnings) {
    skv_rules* r = nullptr;
    char err[1024] = {0};
    const int rc = skv_rules_from_json(text.data(), text.size(), &r, err, sizeof(err));
    b200::check(rc, std::string(err));
    if (warnings)
      for (size_t i = 0; i < skv_rules_warning_count(r); ++i) warnings->emplace_back(skv_rules_warning(r, i));
    return std::shared_ptr<const CompiledRuleSet>(new CompiledRuleSet(r));
  }

  static std::shared_ptr<const CompiledRuleSet> defaults() {
    skv_rules* r = nullptr;
    b200::check(skv_rules_default(&r), "default rules");
    return std::shared_ptr<const CompiledRuleSet>(new CompiledRuleSet(r));
  }

  ~CompiledRuleSet() {
    if (ctx_) skv_destroy(ctx_);
    skv_rules_free(r_);
  }
  CompiledRuleSet(const CompiledRuleSet&) = delete;
  CompiledRuleSet& operator=(const CompiledRuleSet&) = delete;

  // detection.hpp:148-170, on the device: sensitive iff some enabled rule matches; categories of
  // the hit rules in rule order, de-duplicated
  DetectionVerdict scan(std::string_view text) const {
    std::vector<uint32_t> mask(words(), 0);
    {
      std::lock_guard lk(mu_);
      ensure_ctx();
      b200::check(skv_tier1_scan(ctx_, text.data(), text.size(), mask.data()), ctx_);
    }
    return verdict_of(mask.data(), 1);
  }

  // scan() of many independent texts in one device launch (a pipeline drain)
  std::vector<DetectionVerdict> scan_batch(const std::vector<std::string_view>& texts) const {
    std::vector<uint64_t> off(texts.size() + 1, 0);
    for (size_t i = 0; i < texts.size(); ++i) off[i + 1] = off[i] + texts[i].size();
    std::string flat;
    flat.reserve(off.back());
    for (const auto& t : texts) flat.append(t.data(), t.size());
    std::vector<uint32_t> masks(texts.size() * words(), 0);  // word-major
    {
      std::lock_guard lk(mu_);
      ensure_ctx();
      b200::check(skv_tier1_scan_batch(ctx_, flat.data(), off.data(), static_cast<uint32_t>(texts.size()),
                                       masks.data()),
                  ctx_);
    }
    std::vector<DetectionVerdict> out;
    out.reserve(texts.size());
    for (size_t i = 0; i < texts.size(); ++i) out.push_back(verdict_of(masks.data() + i, texts.size()));
    return out;
  }

  size_t size() const { return skv_rules_count(r_); }
  uint64_t version() const { return skv_rules_version(r_); }
  const skv_rules* handle() const { return r_; }

 private:
  explicit CompiledRuleSet(skv_rules* r) : r_(r) {}

  void ensure_ctx() const {
    if (ctx_) return;
    skv_config c;
    skv_config_default(&c);
    c.block_tokens = 16;
    c.window_tokens = 0;
    c.index_capacity = 1024;
    c.max_prompts = 1;
    c.max_tokens = 1 << 12;
    c.max_window_entries = 1;
    c.max_users = 16;
    b200::check(skv_create(&c, &ctx_), nullptr);
    b200::check(skv_set_rules(ctx_, r_), ctx_);
  }

  // detection.hpp:160-169: categories of the hit rules in rule order, de-duplicated
  uint32_t words() const { return skv_rules_mask_words(r_); }

  // mask word w of this verdict at mask[w * stride]
  DetectionVerdict verdict_of(const uint32_t* mask, size_t stride) const {
    DetectionVerdict v;
    v.tier = 1;
    std::vector<bool> hit(size(), false);
    bool any = false;
    for (uint32_t j = 0; j < skv_rules_enabled_count(r_); ++j)
      if (mask[(j / 32) * stride] >> (j % 32) & 1u) hit[skv_rules_enabled_rule(r_, j)] = any = true;
    for (uint32_t i = 0; i < size(); ++i) {
      if (!hit[i]) continue;
      const char* cat = nullptr;
      skv_rules_info(r_, i, nullptr, &cat, nullptr, nullptr);
      bool dup = false;
      for (const auto& c : v.categories) dup |= c == cat;
      if (!dup) v.categories.emplace_back(cat);
    }
    v.sensitive = any;
    v.score = v.sensitive ? 1.0 : 0.0;
    v.escalate = !v.sensitive;
    return v;
  }

  skv_rules* r_ = nullptr;
  mutable std::mutex mu_;
  mutable skv_ctx* ctx_ = nullptr;  // the device scanner of this snapshot (created on first scan)
};

// detection.hpp:185-204
inline std::vector<PatternRule> default_pattern_rules() {
  auto d = CompiledRuleSet::defaults();
  std::vector<PatternRule> out;
  for (uint32_t i = 0; i < d->size(); ++i) {
    const char *id = nullptr, *cat = nullptr;
    int kind = 0, en = 1;
    skv_rules_info(d->handle(), i, &id, &cat, &kind, &en);
    PatternRule r;
    r.rule_id = id;
    r.category = cat;
    r.kind = kind ? PatternRule::Kind::ExactBlacklist : PatternRule::Kind::Regex;
    r.enabled = en != 0;
    out.push_back(r);  // (the pattern text stays inside the compiled set)
  }
  return out;
}

// detection.hpp:208-284
class RuleEngine {
 public:
  RuleEngine() : active_(CompiledRuleSet::defaults()) {}

  std::shared_ptr<const CompiledRuleSet> active() const {
    std::lock_guard lk(mu_);
    return active_;
  }

  DetectionVerdict tier1_scan(std::string_view text) const { return active()->scan(text); }
  // tier1_scan of many texts against one snapshot (one device launch)
  std::vector<DetectionVerdict> tier1_scan_batch(const std::vector<std::string_view>& texts) const {
    return active()->scan_batch(texts);
  }

  // ParseError / CompileError; on failure the previous set stays active
  std::shared_ptr<const CompiledRuleSet> load_rules_json(const nlohmann::json& j,
                                                         std::vector<std::string>* warnings = nullptr) {
    if (!j.is_object()) throw ParseError("pattern config: top level must be an object");
    auto compiled = CompiledRuleSet::from_json_text(j.dump(), warnings);
    std::lock_guard lk(mu_);
    active_ = compiled;
    return compiled;
  }

  std::shared_ptr<const CompiledRuleSet> load_rules(const std::string& path,
                                                    std::vector<std::string>* warnings = nullptr) {
    std::ifstream in(path);
    if (!in) throw ConfigError("cannot open pattern config: " + path);
    nlohmann::json j;
    try {
      in >> j;
    } catch (const nlohmann::json::exception& e) {
      throw ParseError(std::string("pattern config: ") + e.what());
    }
    return load_rules_json(j, warnings);
  }

  std::shared_ptr<const CompiledRuleSet> reload_rules(const std::string& path,
                                                      std::vector<std::string>* warnings = nullptr) {
    return load_rules(path, warnings);
  }

 private:
  mutable std::mutex mu_;
  std::shared_ptr<const CompiledRuleSet> active_;
};


// ---------------------------------------------------------------------------------------------
// Tier-2/3 detectors (detection.hpp:286-416).  Mocks of out-of-process models: a seeded stream per
// detector, consumed in classification order, so a fixed (seed, input order) reproduces the
// reference's verdicts bit for bit.
// ---------------------------------------------------------------------------------------------

// detection.hpp:291-295 (ground truth of one block, from the workload generator)
struct BlockTruth {
  bool sensitive_alone = false;
  bool sensitive_with_context = false;
  std::vector<std::string> categories;
};

// detection.hpp:297-307
struct LatencyModel {
  enum class Kind : uint8_t { Constant, Lognormal } kind = Kind::Constant;
  double value_ms = 0.0;
  double mu = 0.0;
  double sigma = 0.0;
  double sample(SplitMix64& rng) const { return kind == Kind::Constant ? value_ms : std::exp(mu + sigma * rng.next_normal()); }
};

// detection.hpp:309-316
struct DetectorSpec {
  int tier = 2;
  enum class Mode : uint8_t { Oracle, MockWithFNR, External } mode = Mode::Oracle;
  double false_negative_rate = 0.0;
  double false_positive_rate = 0.0;
  LatencyModel latency;
  uint64_t seed = 0;
};

// detection.hpp:318-323
struct BlockInput {
  uint64_t block_id = 0;
  std::string text;
  std::vector<std::string> history;
  BlockTruth truth;
};

// detection.hpp:328-340: the transport-agnostic client of an external detector (the subprocess
// transport of external_detector.hpp is outside the admission path; any client plugs in here)
class ExternalDetectorClient {
 public:
  struct Reply {
    bool sensitive = false;
    double score = 0.0;
    std::vector<std::string> categories;
  };
  virtual ~ExternalDetectorClient() = default;
  virtual Reply request(uint64_t block_id, std::string_view text, const std::vector<std::string>& history) = 0;
};

// detection.hpp:351-416
class Detector {
 public:
  explicit Detector(DetectorSpec spec, std::shared_ptr<ExternalDetectorClient> external = nullptr)
      : spec_(spec), verdict_rng_(spec.seed), latency_rng_(derive_seed(spec.seed, 0x17)), ext_(std::move(external)) {}

  const DetectorSpec& spec() const { return spec_; }
  double sample_latency() { return spec_.latency.sample(latency_rng_); }

  DetectionVerdict classify(const BlockInput& in, double current_threshold) {
    DetectionVerdict v;
    v.tier = spec_.tier;
    if (spec_.mode == DetectorSpec::Mode::External) {
      if (!ext_) throw DetectorUnavailable("external detector not attached");
      const auto r = ext_->request(in.block_id, in.text, in.history);
      v.sensitive = r.sensitive;
      v.score = r.score;
      v.categories = r.categories;
    } else {
      // tier >= 3 with history judges the context-aware truth (detection.hpp:398-401)
      const bool truth = (spec_.tier >= 3 && !in.history.empty()) ? in.truth.sensitive_with_context
                                                                   : in.truth.sensitive_alone;
      if (spec_.mode == DetectorSpec::Mode::Oracle) {
        v.sensitive = truth;
        v.score = 1.0;
      } else {
        const double u = verdict_rng_.next_double();
        v.sensitive = truth ? u >= spec_.false_negative_rate : u < spec_.false_positive_rate;
        if (v.sensitive) {
          v.score = 1.0 - spec_.false_negative_rate;
        } else {  // benign confidence: U[0.1, 0.6) for context-only secrets, else U[0.5, 1)
          const double w = verdict_rng_.next_double();
          const bool context_only = in.truth.sensitive_with_context && !in.truth.sensitive_alone;
          v.score = context_only ? 0.1 + 0.5 * w : 0.5 + 0.5 * w;
        }
      }
      if (v.sensitive && !in.truth.categories.empty()) v.categories = in.truth.categories;
    }
    v.escalate = !v.sensitive && v.score < current_threshold;
    return v;
  }

 private:
  DetectorSpec spec_;
  SplitMix64 verdict_rng_;
  SplitMix64 latency_rng_;
  std::shared_ptr<ExternalDetectorClient> ext_;
};

// detection.hpp:422-449 (adaptive thresholding)
struct ThresholdState {
  double base_threshold = 0.52;
  double current_threshold = 0.52;
  double load_factor = 0.0;
  enum class Alert : uint8_t { Normal, Elevated } alert_level = Alert::Normal;
};

inline ThresholdState adjust_threshold(ThresholdState state, double load, uint64_t recent_alerts, double k_load = 0.05,
                                       double k_alert = 0.02, double t_min = 0.1) {
  if (load < 0) throw Error("adjust_threshold: load must be non-negative");
  const double t = state.base_threshold - k_load * std::max(0.0, load - 1.0) - k_alert * static_cast<double>(recent_alerts);
  state.current_threshold = std::min(state.base_threshold, std::max(t_min, t));
  state.load_factor = load;
  state.alert_level = recent_alerts ? ThresholdState::Alert::Elevated : ThresholdState::Alert::Normal;
  return state;
}

// ---------------------------------------------------------------------------------------------
// Asynchronous classification pipeline (detection.hpp:442-649)
// ---------------------------------------------------------------------------------------------

struct PendingBlock {
  uint64_t block_id = 0;
  NodeRef node = nullptr;  // null for standalone classification runs
  uint32_t span_tokens = 0;
  std::string text;
  std::vector<std::string> history;
  BlockTruth truth;
  double enqueue_ms = 0.0;
};

struct ClassificationOutcome {
  uint64_t block_id = 0;
  NodeRef node = nullptr;
  uint32_t span_tokens = 0;
  SensitivityLabel final_label = SensitivityLabel::Private;
  int resolved_tier = 1;
  double total_latency_ms = 0.0;
  bool truth_sensitive = false;
  bool detector_unavailable = false;
  std::vector<std::string> categories;
};

struct PipelineConfig {
  size_t queue_capacity = 4096;
  size_t batch_size = 64;
  double base_threshold = 0.52;
  double k_load = 0.05;
  double k_alert = 0.02;
  double t_min = 0.1;
  std::optional<DetectorSpec> tier1_mock;  // replaces the rule engine when set
  DetectorSpec tier2{};
  DetectorSpec tier3{};
};

struct PipelineCounters {
  uint64_t enqueued = 0;
  uint64_t saturation_drops = 0;
  uint64_t tier_invocations[3] = {0, 0, 0};
  uint64_t resolved_by_tier[3] = {0, 0, 0};
  uint64_t finalized_public = 0;
  uint64_t finalized_private = 0;
  uint64_t detector_unavailable = 0;
};

// Tier-1 -> (escalate) Tier-2 -> (escalate) Tier-3 per block; the first sensitive verdict finalizes
// Private, a block is Public only when no tier flags it.  A drain takes the queued blocks it will
// classify and scans all of them with one device launch of the active rule snapshot (the rule
// verdict depends on the text alone, so batching it is exact); the mocks and the sink then run per
// block in queue order, as in the reference.
class DetectionPipeline {
 public:
  using Sink = std::function<void(const ClassificationOutcome&)>;

  DetectionPipeline(PipelineConfig cfg, RuleEngine* rules, Sink sink,
                    std::shared_ptr<ExternalDetectorClient> tier2_ext = nullptr,
                    std::shared_ptr<ExternalDetectorClient> tier3_ext = nullptr)
      : cfg_(cfg),
        rules_(rules),
        sink_(std::move(sink)),
        tier1_(cfg.tier1_mock ? std::make_unique<Detector>(*cfg.tier1_mock) : nullptr),
        tier2_(cfg.tier2, std::move(tier2_ext)),
        tier3_(cfg.tier3, std::move(tier3_ext)) {
    threshold_.base_threshold = threshold_.current_threshold = cfg.base_threshold;
  }

  // detection.hpp:507-516: false (a saturation drop; the block stays PendingPrivate) when full
  bool enqueue(PendingBlock block) {
    std::lock_guard lk(mu_);
    if (queue_.size() >= cfg_.queue_capacity) {
      ++counters_.saturation_drops;
      return false;
    }
    ++counters_.enqueued;
    queue_.push_back(std::move(block));
    return true;
  }

  // detection.hpp:520-536: classifies up to max_blocks (default: the batch size) queued blocks
  size_t drain(size_t max_blocks = 0) {
    if (max_blocks == 0) max_blocks = cfg_.batch_size;
    size_t done = 0;
    while (done < max_blocks) {
      std::vector<PendingBlock> batch;
      {
        std::lock_guard lk(mu_);
        while (!queue_.empty() && done + batch.size() < max_blocks) {
          batch.push_back(std::move(queue_.front()));
          queue_.pop_front();
        }
      }
      if (batch.empty()) break;
      std::vector<DetectionVerdict> tier1;
      if (!tier1_ && rules_) {
        std::vector<std::string_view> texts;
        texts.reserve(batch.size());
        for (const auto& b : batch) texts.emplace_back(b.text);
        tier1 = rules_->tier1_scan_batch(texts);
      }
      for (size_t i = 0; i < batch.size(); ++i) {
        ClassificationOutcome out = classify(batch[i], tier1.empty() ? nullptr : &tier1[i]);
        if (sink_) sink_(out);
        ++done;
      }
    }
    return done;
  }

  size_t queue_size() const {
    std::lock_guard lk(mu_);
    return queue_.size();
  }

  void update_threshold(double load, uint64_t recent_alerts) {
    std::lock_guard lk(mu_);
    threshold_ = adjust_threshold(threshold_, load, recent_alerts, cfg_.k_load, cfg_.k_alert, cfg_.t_min);
  }

  ThresholdState threshold() const {
    std::lock_guard lk(mu_);
    return threshold_;
  }

  const PipelineCounters& counters() const { return counters_; }
  const PipelineConfig& config() const { return cfg_; }

 private:
  // detection.hpp:559-631
  ClassificationOutcome classify(const PendingBlock& blk, const DetectionVerdict* rule_verdict) {
    ClassificationOutcome out;
    out.block_id = blk.block_id;
    out.node = blk.node;
    out.span_tokens = blk.span_tokens;
    out.truth_sensitive = blk.truth.sensitive_with_context || blk.truth.sensitive_alone;
    const double thr = threshold().current_threshold;
    const BlockInput in{blk.block_id, blk.text, blk.history, blk.truth};

    ++counters_.tier_invocations[0];
    DetectionVerdict v1;
    if (tier1_) {
      v1 = tier1_->classify(in, thr);
      v1.tier = 1;
      v1.escalate = !v1.sensitive;
      out.total_latency_ms += tier1_->sample_latency();
    } else {
      v1 = rule_verdict ? *rule_verdict : rules_->tier1_scan(blk.text);
    }
    if (v1.sensitive) return finalize(out, SensitivityLabel::Private, 1, std::move(v1.categories));

    Detector* const later[2] = {&tier2_, &tier3_};
    for (int t = 2; t <= 3; ++t) {
      ++counters_.tier_invocations[t - 1];
      DetectionVerdict v;
      try {
        v = later[t - 2]->classify(in, thr);
        out.total_latency_ms += later[t - 2]->sample_latency();
      } catch (const DetectorUnavailable&) {
        out.detector_unavailable = true;
        ++counters_.detector_unavailable;
        return finalize(out, SensitivityLabel::Private, t, {});
      }
      if (t == 3)
        return finalize(out, v.sensitive ? SensitivityLabel::Private : SensitivityLabel::Public, 3,
                        std::move(v.categories));
      if (v.sensitive) return finalize(out, SensitivityLabel::Private, 2, std::move(v.categories));
      if (!v.escalate) return finalize(out, SensitivityLabel::Public, 2, {});
    }
    return out;  // unreachable
  }

  ClassificationOutcome& finalize(ClassificationOutcome& out, SensitivityLabel label, int tier,
                                  std::vector<std::string> categories) {
    out.final_label = label;
    out.resolved_tier = tier;
    out.categories = std::move(categories);
    ++counters_.resolved_by_tier[tier - 1];
    if (label == SensitivityLabel::Public)
      ++counters_.finalized_public;
    else
      ++counters_.finalized_private;
    return out;
  }

  PipelineConfig cfg_;
  RuleEngine* rules_;
  Sink sink_;
  std::unique_ptr<Detector> tier1_;
  Detector tier2_;
  Detector tier3_;
  mutable std::mutex mu_;
  std::deque<PendingBlock> queue_;
  ThresholdState threshold_;
  PipelineCounters counters_;
};

// detection.hpp:667-676: the production sink applies an outcome to the (device) index -- Public
// promotions never propagate, private finalizations propagate to descendants; the audit byte
// records the tiers a promoted block passed
inline DetectionPipeline::Sink make_index_sink(RadixCacheIndex& index) {
  return [&index](const ClassificationOutcome& out) {
    if (!out.node) return;
    uint8_t audit = 0;
    for (int t = 1; t <= out.resolved_tier; ++t) audit |= static_cast<uint8_t>(1u << (t - 1));
    const bool priv = out.final_label != SensitivityLabel::Public;
    index.resolve_block(out.node, out.span_tokens, out.final_label, priv, priv ? 0 : audit);
  };
}

}  // namespace safekv
