// detection.hpp -- drop-in facade of the reference's Tier-1 rule engine (proj/include/safekv/
// detection.hpp:28-284): PatternRule, DetectionVerdict, CompiledRuleSet (an immutable compiled
// snapshot) and the hot-reloadable RuleEngine.  Rule sets compile on the host into the one search
// DFA the device scans (skv_rules_*); scan() runs on the device (skv_tier1_scan) against the
// snapshot it is called on.  The Tier-2/3 detectors and the asynchronous pipeline of the reference
// header are out of the admission path.
#pragma once

#include <fstream>
#include <memory>
#include <mutex>
#include <nlohmann/json.hpp>
#include <sstream>
#include <string>
#include <string_view>
#include <vector>

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
    uint32_t mask = 0;
    {
      std::lock_guard lk(mu_);
      if (!ctx_) {
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
      b200::check(skv_tier1_scan(ctx_, text.data(), text.size(), &mask), ctx_);
    }
    DetectionVerdict v;
    v.tier = 1;
    std::vector<bool> hit(size(), false);
    for (uint32_t j = 0; j < skv_rules_enabled_count(r_); ++j)
      if (mask >> j & 1u) hit[skv_rules_enabled_rule(r_, j)] = true;
    for (uint32_t i = 0; i < size(); ++i) {
      if (!hit[i]) continue;
      const char* cat = nullptr;
      skv_rules_info(r_, i, nullptr, &cat, nullptr, nullptr);
      bool dup = false;
      for (const auto& c : v.categories) dup |= c == cat;
      if (!dup) v.categories.emplace_back(cat);
    }
    v.sensitive = mask != 0;
    v.score = v.sensitive ? 1.0 : 0.0;
    v.escalate = !v.sensitive;
    return v;
  }

  size_t size() const { return skv_rules_count(r_); }
  uint64_t version() const { return skv_rules_version(r_); }
  const skv_rules* handle() const { return r_; }

 private:
  explicit CompiledRuleSet(skv_rules* r) : r_(r) {}
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

}  // namespace safekv
