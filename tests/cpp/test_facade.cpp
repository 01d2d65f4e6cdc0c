// test_facade.cpp -- the reference's unit tests for the admission path, restated against
// the C++ facade (include/safekv_b200/safekv.hpp) so they read like
// proj/tests/unit/test_{detection,cache_index,monitor,core}.cpp.  Needs an sm_100 GPU;
// built and run by tests/test_gpu_facade.py.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "safekv_b200/safekv.hpp"

using namespace safekv_b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(x)                                                             \
  do {                                                                       \
    ++g_checks;                                                              \
    if (!(x)) {                                                              \
      ++g_fail;                                                              \
      std::fprintf(stderr, "%s:%d CHECK failed: %s\n", __FILE__, __LINE__, #x); \
    }                                                                        \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static skv_config small_cfg(uint32_t B) {
  skv_config c;
  skv_config_default(&c);
  c.block_tokens = B;
  c.window_tokens = 0;
  c.index_capacity = 1 << 12;
  c.max_prompts = 256;
  c.max_tokens = 1 << 14;
  c.max_window_entries = 1 << 10;
  return c;
}

int main() {
  AdmissionIndex idx;  // defaults: B = 16, W = 32

  // test_detection.cpp:33-42
  {
    DetectionVerdict v = idx.tier1_scan("my ssn is 123-45-6789");
    CHECK(v.sensitive);
    CHECK(v.tier == 1);
    CHECK(v.score == 1.0);
    CHECK(!v.categories.empty() && v.categories[0] == "Identity Information");
    CHECK(!v.escalate);
  }
  // :44-50
  {
    DetectionVerdict v = idx.tier1_scan("the weather is nice");
    CHECK(!v.sensitive);
    CHECK(v.escalate);
    CHECK(v.categories.empty());
  }
  // :52-57 blacklist terms match whole tokens only
  CHECK(idx.tier1_scan("status of PROJECT-TITAN today").sensitive);
  CHECK(idx.tier1_scan("see (PROJECT-TITAN).").sensitive);
  CHECK(!idx.tier1_scan("PROJECT-TITANIC is something else").sensitive);
  // :59-77 every default rule fires on its template family
  {
    const std::vector<std::pair<std::string, std::string>> samples = {
        {"my ssn is 987-65-4321", "Identity Information"},
        {"call me at (415) 555-0134", "Basic Information"},
        {"email me at user99@mail01.com", "Basic Information"},
        {"server at 10.4.77.3", "System/Network Identification"},
        {"card number 4111-1111-1111-1111", "Financial Info"},
        {"account number 48392057", "Financial Info"},
        {"device mac 0a:1b:2c:3d:4e:5f", "Hardware Device Information"},
        {"imei 490154203237518", "Hardware Device Information"},
    };
    for (const auto& [text, cat] : samples) {
      DetectionVerdict v = idx.tier1_scan(text);
      bool has = false;
      for (const auto& c : v.categories) has = has || c == cat;
      CHECK(v.sensitive && has);
    }
  }
  // :79-108 rule loading validates and rejects atomically
  {
    std::string good =
        R"({"version":2,"rules":[{"rule_id":"a","category":"X","kind":"regex","pattern":"foo"},)"
        R"({"rule_id":"b","category":"Y","kind":"blacklist","pattern":"BAR"},)"
        R"({"rule_id":"c","category":"Z","kind":"regex","pattern":"qu+x"}]})";
    auto set = idx.load_rules_json(good);
    CHECK(set->size() == 3);
    CHECK(set->version() == 2);
    CHECK(idx.tier1_scan("a foo b").sensitive);
    std::string bad = good;
    bad.replace(bad.find("\"blacklist\",\"pattern\":\"BAR\""), 27, "\"regex\",\"pattern\":\"(\"");
    bool named = false;
    try {
      idx.load_rules_json(bad);
    } catch (const CompileError& e) {
      named = std::string(e.what()).find("'b'") != std::string::npos;
    }
    CHECK(named);
    CHECK(idx.active()->version() == 2);  // previous set still active
    std::vector<std::string> warnings;
    idx.load_rules_json(R"({"version":3,"surprise":1,"rules":[]})", &warnings);
    CHECK(warnings.size() == 1 && warnings[0].find("surprise") != std::string::npos);
    // :110-118 disabled rules do not match
    idx.load_rules_json(
        R"({"version":1,"rules":[{"rule_id":"off","category":"X","kind":"regex","pattern":"danger","enabled":false}]})");
    CHECK(!idx.tier1_scan("danger zone").sensitive);
    // a library of more than 32 enabled rules (several mask words): a verdict from any word, the
    // categories in rule order (detection.hpp:160-169)
    std::string wide = R"({"version":9,"rules":[)";
    for (int i = 0; i < 70; ++i)
      wide += std::string(i ? "," : "") + R"({"rule_id":"w)" + std::to_string(i) + R"(","category":"C)" +
              std::to_string(i % 7) + R"(","kind":"regex","pattern":"tok)" + std::to_string(i) + R"(x"})";
    wide += "]}";
    auto ws = idx.load_rules_json(wide);
    CHECK(ws->mask_words() == 3);
    DetectionVerdict v65 = idx.tier1_scan("a tok65x b");
    CHECK(v65.sensitive && v65.categories.size() == 1 && v65.categories[0] == "C2");
    DetectionVerdict v2 = idx.tier1_scan("tok69x tok3x tok40x");  // rules 3 (C3), 40 (C5), 69 (C6)
    CHECK(v2.sensitive && v2.categories.size() == 3 && v2.categories[0] == "C3" && v2.categories[1] == "C5" &&
          v2.categories[2] == "C6");
    CHECK(!idx.tier1_scan("tok70x").sensitive);
  }
  // test_core.cpp:31-45 digests are structural
  {
    TokenSeq s{1, 2, 3, 250, 7};
    TokenSeq t = s;
    CHECK(idx.token_seq_digest(s) == idx.token_seq_digest(t));
    t[2] ^= 1;
    CHECK(idx.token_seq_digest(s) != idx.token_seq_digest(t));
  }

  const UserId alice{1}, bob{2};
  // test_cache_index.cpp:103-109 private nodes are invisible to non-creators
  // (block-granular: B = 4, no rules -> labels from the rule tier are Public, so the
  // private label comes from a rule hit: "PROJECT-TITAN" lands in the first window)
  {
    skv_config c = small_cfg(4);
    c.window_tokens = 16;
    AdmissionIndex ix(&c);
    std::string text = "PROJECT-TITAN x";
    TokenSeq seq(text.begin(), text.end());
    ix.insert(seq, alice, OwnerClass::Customer);
    CHECK(ix.match_prefix(seq, bob).matched_tokens == 0);
    CHECK(ix.match_prefix(seq, alice).matched_tokens == (seq.size() / 4) * 4);
    // a public sequence is shared with everyone
    std::string pub = "the weather is nice today";
    TokenSeq ps(pub.begin(), pub.end());
    ix.insert(ps, alice, OwnerClass::Customer);
    CHECK(ix.match_prefix(ps, bob).matched_tokens == (ps.size() / 4) * 4);
    // partial coverage: the shared prefix matches up to the divergence (block granular)
    TokenSeq q(ps.begin(), ps.begin() + 9);
    q.push_back('Z');
    q.push_back('Z');
    q.push_back('Z');
    CHECK(ix.match_prefix(q, bob).matched_tokens == 8);
  }
  // test_monitor.cpp:101-120 suspicious burst downgrades a customer block and hides the subtree
  // test_monitor.cpp:135-153 business blocks are restricted
  for (OwnerClass owner : {OwnerClass::Customer, OwnerClass::Business}) {
    AdmissionIndex ix(&(const skv_config&)small_cfg(4));
    TokenSeq two{1, 2, 3, 4, 5, 6, 7, 8}, one{1, 2, 3, 4};
    ix.insert(two, alice, owner);
    ix.epoch_pass();
    std::vector<AdmissionIndex::Request> prev(20, AdmissionIndex::Request{&one, alice, owner});
    ix.admit(prev);  // previous window: 20 hits by one user
    ix.commit();
    ix.epoch_pass();
    std::vector<UserId> burst{{10}, {11}, {12}, {13}, {14}, {15}, {10}, {11}};
    std::vector<AdmissionIndex::Request> cur;
    for (auto& u : burst) cur.push_back(AdmissionIndex::Request{&one, u, owner});
    ix.admit(cur);
    ix.commit();
    auto ev = ix.epoch_pass();
    CHECK(ev.size() == 1);
    if (ev.size() == 1) {
      CHECK(ev[0].action == (owner == OwnerClass::Customer ? AnomalyAction::DowngradeToPrivate
                                                           : AnomalyAction::Restrict));
      CHECK(std::fabs(ev[0].entropy_prev - 1.0 / 20.0) < 1e-12);
      CHECK(std::fabs(ev[0].entropy_now - 0.75) < 1e-12);
      CHECK(ev[0].owner_class == owner);
    }
    CHECK(ix.match_prefix(two, bob).matched_tokens == 0);    // downgraded block + child hidden
    CHECK(ix.match_prefix(two, alice).matched_tokens == 8);  // creator still sees both
  }
  // test_monitor.cpp:122-133 historically broad reuse is not suspicious
  {
    AdmissionIndex ix(&(const skv_config&)small_cfg(4));
    TokenSeq one{1, 2, 3, 4};
    ix.insert(one, alice, OwnerClass::Customer);
    ix.epoch_pass();
    std::vector<UserId> us;
    for (uint64_t u = 1; u <= 12; ++u) us.push_back(UserId{u});
    std::vector<AdmissionIndex::Request> r;
    for (auto& u : us) r.push_back(AdmissionIndex::Request{&one, u});
    ix.admit(r);
    ix.commit();
    ix.epoch_pass();  // u_pre = 12
    std::vector<UserId> us2;
    for (uint64_t u = 20; u < 26; ++u) us2.push_back(UserId{u});
    r.clear();
    for (auto& u : us2) r.push_back(AdmissionIndex::Request{&one, u});
    ix.admit(r);
    ix.commit();
    CHECK(ix.epoch_pass().empty());
  }
  // CapacityExhausted when the index is full (cache_index.hpp:801-806 analogue)
  {
    skv_config c = small_cfg(4);
    c.index_capacity = 1024;
    AdmissionIndex ix(&c);
    bool hit = false;
    for (uint32_t k = 0; k < 64 && !hit; ++k) {
      TokenSeq s;
      for (uint32_t i = 0; i < 64; ++i) s.push_back(k * 1000 + i + 1);
      hit = throws<CapacityExhausted>([&] { ix.insert(s, alice, OwnerClass::Customer); });
    }
    CHECK(hit);
  }
  // test_serving_sim.cpp:36-67 (block-granular: public blocks of 8 tokens, HBM)
  {
    AdmissionIndex ix(&(const skv_config&)small_cfg(8));
    ix.set_cost_model(AdmissionIndex::CostModel{});
    TokenSeq text(96, 'q');
    ix.admit({AdmissionIndex::Request{&text, UserId{1}}});
    auto cold = ix.served(1);
    CHECK(std::fabs(cold.ttft_ms[0] - 106.0) < 1e-12);  // t_base 10 + 1 ms * 96 (cold cache)
    ix.commit();
    ix.admit({AdmissionIndex::Request{&text, UserId{2}}});
    auto hit = ix.served(1);
    CHECK(std::fabs(hit.ttft_ms[0] - 10.0) < 1e-12);  // full public HBM hit: base time only
    CHECK(hit.inter_tokens[0] == 96 && hit.intra_tokens[0] == 0);
    ix.commit();
    double prev = 1e18;
    for (size_t matched = 8; matched <= 96; matched += 8) {  // strictly decreasing with the match
      TokenSeq probe(text.begin(), text.begin() + matched);
      probe.resize(96, '!');
      ix.admit({AdmissionIndex::Request{&probe, UserId{100 + matched}}});
      double t = ix.served(1).ttft_ms[0];
      CHECK(t < prev);
      prev = t;
    }
    // test_serving_sim.cpp:258-267 CostModel::validate
    AdmissionIndex::CostModel broken;
    broken.c_prefill_ms = 0.1;
    CHECK(throws<ConfigError>([&] { ix.set_cost_model(broken); }));
    AdmissionIndex::CostModel neg;
    neg.tier_penalty_ms[1] = 0.9;
    neg.tier_penalty_ms[2] = 0.5;
    CHECK(throws<ConfigError>([&] { ix.set_cost_model(neg); }));
  }
  // eviction (cache_index.hpp:281-292): oldest access epoch first; an evicted key is gone
  // for lookups until it is inserted again
  {
    skv_config cfg = small_cfg(4);
    AdmissionIndex ix(&cfg);
    ix.enable_eviction();
    const std::string a = "aaaabbbbccccdddd", b = "eeeeffffgggghhhh";
    TokenSeq sa(a.begin(), a.end()), sb(b.begin(), b.end());
    CHECK(ix.insert(sa, UserId{1}, OwnerClass::Customer) == 4);
    ix.epoch_pass();  // sa's blocks keep the older access epoch
    CHECK(ix.insert(sb, UserId{2}, OwnerClass::Customer) == 4);
    auto victims = ix.evict(4);
    CHECK(victims.size() == 4);
    CHECK(ix.entry_count() == 4);
    CHECK(ix.match_prefix(sa, UserId{9}).matched_tokens == 0);   // evicted
    CHECK(ix.match_prefix(sb, UserId{9}).matched_tokens == 16);  // kept
    CHECK(ix.insert(sa, UserId{1}, OwnerClass::Customer) == 4);  // re-inserted as fresh entries
    CHECK(ix.match_prefix(sa, UserId{9}).matched_tokens == 16);
    CHECK(throws<CapacityExhausted>([&] { ix.evict(100); }));
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
