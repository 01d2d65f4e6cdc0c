// rules.hpp -- host-side Tier-1 rule compiler: rule JSON -> one multi-pattern search DFA.
//
// Replaces the per-window work of CompiledRuleSet::scan (reference
// include/safekv/detection.hpp:148-170: one std::regex_search per enabled regex rule
// plus a whole-token TokenTrie pass, :79-100) by a single table-driven automaton that
// the device scans in one pass per window.  The front end mirrors libstdc++'s
// ECMAScript scanner/compiler (GCC 13.3, the reference's regex implementation) so the
// same patterns are accepted and the same byte strings match; constructs a DFA cannot
// express (back-references, lookahead) are rejected with CompileError -- a documented
// divergence (DESIGN.md section "Rule tier").
#pragma once

#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace skv {

// Error taxonomy mirrors safekv::Error subclasses (reference core.hpp:19-59).
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
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

// reference detection.hpp:28-34
struct PatternRule {
  std::string rule_id;
  std::string category;
  bool blacklist = false;  // Kind::ExactBlacklist
  std::string pattern;
  bool enabled = true;
};

struct RuleSetSpec {
  uint64_t version = 0;
  std::vector<PatternRule> rules;
  std::vector<std::string> warnings;
};

// reference detection.hpp:185-204 (the nine shipped rules).
std::vector<PatternRule> default_pattern_rules();

// reference RuleEngine::load_rules_json / parse_rule (detection.hpp:222-280).
// Throws ParseError.  Unknown fields become warnings.
RuleSetSpec parse_rules_json(const std::string& json);

// Compiled search automaton.  Transition on byte class c from state s emits the
// rule mask acc[s*(C+1)+c] (rules whose match ends at the position BEFORE consuming
// the symbol, assertions evaluated with the symbol as look-ahead) and moves to
// next[s*C+c].  Column C of acc is the end-of-text (EOS) transition.
// Bit j of a mask = j-th ENABLED rule (rule_index[j] is its position in the list).
struct DfaTables {
  uint32_t n_states = 0;
  uint32_t n_classes = 0;  // byte classes, EOS excluded
  uint32_t start = 0;
  uint8_t class_map[256] = {};
  std::vector<uint16_t> next;        // n_states * n_classes
  std::vector<uint32_t> acc;         // n_states * (n_classes + 1)
  std::vector<uint32_t> rule_index;  // enabled-rule ordinal -> rule list position
  uint32_t nfa_states = 0;           // diagnostics
  uint32_t dfa_states_unminimized = 0;
};

// reference CompiledRuleSet::compile (detection.hpp:120-144): duplicate rule_id and
// bad regex raise CompileError naming the rule.
DfaTables compile_rules(const std::vector<PatternRule>& rules);

// Device rule groups: the enabled rules, in order, cut into consecutive groups of at most
// max_group rules whose automaton satisfies `fits` (the device table limits); each group is
// compiled over the full list with the other rules disabled (so duplicate blacklist terms keep
// the reference's last-writer semantics, detection.hpp:62,157-159).  Group g's mask bit k is the
// (first_bit[g] + k)-th enabled rule.  CompileError if a single rule does not fit.
struct RuleGroups {
  std::vector<DfaTables> groups;
  std::vector<uint32_t> first_bit;
};
RuleGroups compile_rule_groups(const std::vector<PatternRule>& rules, const std::function<bool(const DfaTables&)>& fits,
                               uint32_t max_group = 16);

}  // namespace skv
