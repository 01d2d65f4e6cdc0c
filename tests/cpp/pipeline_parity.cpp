// pipeline_parity.cpp -- one serving-style labeling scenario through the Tier-1/2/3
// DetectionPipeline with the production index sink (detection.hpp:491-676 of the reference).
// TEST INFRASTRUCTURE: the same source is compiled twice --
//   * against the reference's own headers (oracle/Makefile -> oracle/_ref/pipeline_parity_ref), and
//   * against the drop-in facade include/safekv/ + libsafekv_b200.so (tests/test_gpu_pipeline.py),
// and the two transcripts must be identical: every outcome (label, tier, latency, categories), the
// pipeline counters, the threshold trajectory, and what every user then sees in the index (match
// lengths, slowest tier, and the per-token labels the creator sees).
//
// Requests are byte-token texts (ByteVocabulary): a shared prefix from a small pool, then a body
// that may carry a planted secret (sensitive alone: the rule tier sees it unless it is written in a
// form the rules miss) or a context-only secret (sensitive only with the session history, which the
// Tier-3 mock sees).  Each insert's new suffix is one pending block, classified asynchronously in
// drains of varying size under a varying load/alert threshold.
#include <algorithm>
#include <cinttypes>
#include <cstdlib>
#include <memory>
#include <cstdio>
#include <string>
#include <vector>

#include "safekv/cache_index.hpp"
#include "safekv/detection.hpp"

using namespace safekv;

namespace {

struct Req {
  TokenSeq seq;
  UserId user;
};

TokenSeq bytes(const std::string& s) {
  TokenSeq t;
  for (unsigned char c : s) t.push_back(c);
  return t;
}

const char* label_name(SensitivityLabel l) {
  switch (l) {
    case SensitivityLabel::Public: return "Public";
    case SensitivityLabel::PendingPrivate: return "Pending";
    case SensitivityLabel::Private: return "Private";
    case SensitivityLabel::Restricted: return "Restricted";
  }
  return "?";
}

char label_char(SensitivityLabel l) {
  switch (l) {
    case SensitivityLabel::Public: return '.';
    case SensitivityLabel::PendingPrivate: return '?';
    case SensitivityLabel::Private: return 'P';
    case SensitivityLabel::Restricted: return 'R';
  }
  return '!';
}

// a deterministic external detector (the reference's ExternalDetectorClient interface): flags texts
// containing a digit run, and is unavailable for every ninth block
class ScriptedDetector : public ExternalDetectorClient {
 public:
  Reply request(uint64_t block_id, std::string_view text, const std::vector<std::string>& history) override {
    if (block_id % 9 == 0) throw DetectorUnavailable("scripted outage");
    Reply r;
    int run = 0, best = 0;
    for (char c : text) best = std::max(best, run = (c >= '0' && c <= '9') ? run + 1 : 0);
    r.sensitive = best >= 5 && !history.empty();
    r.score = r.sensitive ? 0.9 : 0.3 + 0.05 * static_cast<double>(text.size() % 7);
    if (r.sensitive) r.categories = {"Scripted"};
    return r;
  }
};

}  // namespace

// argv: seed, mode (0: rule tier + Tier-2/3 mocks; 1: Tier-3 is an external client with outages;
// 2: a Tier-1 mock replaces the rule engine)
int main(int argc, char** argv) {
  const uint64_t seed = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 7;
  const int mode = argc > 2 ? std::atoi(argv[2]) : 0;
  SplitMix64 rng(seed);

  RadixCacheIndex index;
  RuleEngine rules;
  PipelineConfig cfg;
  cfg.queue_capacity = 12;  // small: a burst overflows and its blocks stay PendingPrivate
  cfg.batch_size = 5;
  cfg.tier2 = DetectorSpec{2, DetectorSpec::Mode::MockWithFNR, 0.2, 0.05, {}, seed + 11};
  cfg.tier2.latency.kind = LatencyModel::Kind::Lognormal;
  cfg.tier2.latency.mu = 1.0;
  cfg.tier2.latency.sigma = 0.4;
  cfg.tier3 = DetectorSpec{3, DetectorSpec::Mode::MockWithFNR, 0.29, 0.02, {}, seed + 23};
  cfg.tier3.latency.value_ms = 35.0;
  std::shared_ptr<ExternalDetectorClient> ext;
  if (mode == 1) {
    cfg.tier3.mode = DetectorSpec::Mode::External;
    ext = std::make_shared<ScriptedDetector>();
  }
  if (mode == 2) {
    cfg.tier1_mock = DetectorSpec{1, DetectorSpec::Mode::MockWithFNR, 0.5, 0.1, {}, seed + 5};
    cfg.tier1_mock->latency.value_ms = 0.25;
  }

  std::vector<ClassificationOutcome> outcomes;
  auto index_sink = make_index_sink(index);
  DetectionPipeline pipe(
      cfg, &rules,
      [&](const ClassificationOutcome& o) {
        outcomes.push_back(o);
        index_sink(o);
      },
      nullptr, ext);

  const std::vector<std::string> prefixes = {
      "System: you are a helpful banking assistant. ",
      "System: summarise the following support ticket. ",
      "System: translate to French. ",
      "",
  };
  const std::vector<std::string> secrets = {
      "my ssn is 123-45-6789",        "card 4111 1111 1111 1111 expires",
      "email me at jane.doe@example.com", "status of PROJECT-TITAN today",
      "account number 12345678 please",   "call me at (555) 123-4567",
  };
  const std::vector<std::string> fillers = {"the weather is nice ", "please reschedule the meeting ",
                                            "what is the capital of peru ", "list three prime numbers ",
                                            "how do i bake bread "};
  std::vector<Req> reqs;
  uint64_t block_id = 0;
  const int n_req = 160;
  for (int r = 0; r < n_req; ++r) {
    const UserId user{1 + rng.next_below(6)};
    std::string text = prefixes[rng.next_below(prefixes.size())];
    BlockTruth truth;
    std::vector<std::string> history;
    const uint64_t kind = rng.next_below(10);
    text += fillers[rng.next_below(fillers.size())];
    if (kind < 3) {  // a planted secret
      text += secrets[rng.next_below(secrets.size())];
      truth.sensitive_alone = truth.sensitive_with_context = true;
      truth.categories = {"Planted"};
    } else if (kind < 5) {  // context-only: sensitive with the session history
      text += "the code is " + std::to_string(10000 + rng.next_below(90000));
      truth.sensitive_with_context = true;
      truth.categories = {"Financial Info"};
      if (rng.next_below(2)) history = {"my savings account at bankx"};
    } else if (kind == 5) {  // a repeat of an earlier request (structural reuse, no new suffix)
      if (!reqs.empty()) {
        const TokenSeq& prev = reqs[rng.next_below(reqs.size())].seq;
        text.assign(prev.begin(), prev.end() - 1);  // all but the last byte: a prefix of an earlier request
      }
    }
    text += fillers[rng.next_below(fillers.size())];
    Req q{bytes(text), user};
    uint32_t fresh = 0;
    NodeRef node = index.insert(q.seq, user, OwnerClass::Customer, 0, &fresh);
    std::printf("insert %d user %" PRIu64 " len %zu new %u\n", r, user.value, q.seq.size(), fresh);
    if (fresh) {
      PendingBlock b;
      b.block_id = ++block_id;
      b.node = node;
      b.span_tokens = fresh;
      b.text.assign(q.seq.end() - fresh, q.seq.end());
      b.history = history;
      b.truth = truth;
      const bool ok = pipe.enqueue(std::move(b));
      if (!ok) std::printf("  dropped block %" PRIu64 "\n", block_id);
    }
    reqs.push_back(q);
    if (r % 7 == 6) {
      const size_t want = rng.next_below(3) ? 0 : 1 + rng.next_below(12);
      std::printf("drain(%zu) -> %zu\n", want, pipe.drain(want));
    }
    if (r % 23 == 22) {
      pipe.update_threshold(0.5 * static_cast<double>(rng.next_below(9)), rng.next_below(4));
      std::printf("threshold %.17g\n", pipe.threshold().current_threshold);
    }
  }
  while (pipe.drain(0)) {
  }

  for (const auto& o : outcomes) {
    std::printf("outcome %" PRIu64 " span %u %s tier %d lat %.17g truth %d unavail %d cats", o.block_id,
                o.span_tokens, label_name(o.final_label), o.resolved_tier, o.total_latency_ms, o.truth_sensitive,
                o.detector_unavailable);
    for (const auto& c : o.categories) std::printf(" [%s]", c.c_str());
    std::printf("\n");
  }
  const auto& k = pipe.counters();
  std::printf("counters enq %" PRIu64 " drops %" PRIu64 " inv %" PRIu64 "/%" PRIu64 "/%" PRIu64 " res %" PRIu64
              "/%" PRIu64 "/%" PRIu64 " pub %" PRIu64 " priv %" PRIu64 " unavail %" PRIu64 "\n",
              k.enqueued, k.saturation_drops, k.tier_invocations[0], k.tier_invocations[1], k.tier_invocations[2],
              k.resolved_by_tier[0], k.resolved_by_tier[1], k.resolved_by_tier[2], k.finalized_public,
              k.finalized_private, k.detector_unavailable);

  // what the index now shows: every request as seen by every user, and the creator's per-token labels
  for (size_t i = 0; i < reqs.size(); ++i) {
    std::printf("req %zu seen", i);
    for (uint64_t u = 1; u <= 6; ++u) {
      MatchResult m = index.match_prefix(reqs[i].seq, UserId{u});
      std::printf(" %" PRIu64 ":%" PRIu64 "/%d", u, m.matched_tokens, static_cast<int>(m.lowest_tier));
    }
    MatchResult own = index.match_prefix(reqs[i].seq, reqs[i].user);
    std::string labels;
    uint64_t covered = 0;
    for (const auto& n : own.path) {
      const uint64_t take = std::min<uint64_t>(n->span(), own.matched_tokens - covered);
      labels.append(take, label_char(n->label));
      covered += take;
    }
    std::printf(" labels %s\n", labels.c_str());
  }
  return 0;
}
