// cache_index.hpp -- drop-in facade of the reference's RadixCacheIndex (proj/include/safekv/
// cache_index.hpp:26-836) over the B200 device index (include/safekv_b200.h): the same namespace,
// class, method names, argument meanings and exceptions, so a caller compiled against the reference
// header compiles against this one with a type swap.  Every operation runs on the
// device; nothing here computes an index result on the host.
//
// Representation.  The device index is block-granular; the facade
// uses one-token blocks, so matches stay token-granular as in the reference.  A NodeRef names the
// tokens one insert created (the reference's node for that insert: its edge), by the chained keys
// of its blocks; its label is the label of all its blocks, its AccessStats window lives on its
// first block (so a monitor downgrade of the node relabels the node's blocks and everything under
// them, exactly like the reference's subtree relabel).  Differences from the reference:
//  * a NodeRef is a handle, not a CacheNode*: `node->field` reads the device (a snapshot);
//  * node identities follow inserts, not the reference's later edge splits (an insert of a
//    prefix of an existing node returns a one-token node at the prefix end);
//  * node_count() counts device entries (tokens), not radix nodes;
//  * compression and per-node pinning are not provided, and eviction is per block rather than per
//    multi-token radix node, so the facade's TierBudget is bookkeeping only: budgets with
//    insert-time make_room and the evict_or_demote cascade run on the batch path
//    (skv_set_tier_budget).
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "access_stats.hpp"
#include "core.hpp"

namespace safekv {

// cache_index.hpp:26-55
struct TierBudget {
  std::array<uint64_t, 3> capacity_tokens{0, 0, 0};
  std::array<uint64_t, 3> used_tokens{0, 0, 0};

  static TierBudget from_tokens(uint64_t hbm, uint64_t dram, uint64_t ssd) {
    TierBudget b;
    b.capacity_tokens = {hbm, dram, ssd};
    return b;
  }
  static TierBudget from_memory_sizes(uint64_t kv_bytes, uint64_t bytes_per_token, uint64_t dram_tokens = 0,
                                      uint64_t ssd_tokens = 0) {
    if (bytes_per_token == 0) throw ConfigError("bytes_per_token must be positive");
    return from_tokens(kv_bytes / bytes_per_token, dram_tokens, ssd_tokens);
  }
  uint64_t capacity(MemTier t) const { return capacity_tokens[static_cast<size_t>(t)]; }
  uint64_t used(MemTier t) const { return used_tokens[static_cast<size_t>(t)]; }
  uint64_t free_tokens(MemTier t) const { return capacity(t) - used(t); }
  bool can_fit(MemTier t, uint64_t tokens) const { return free_tokens(t) >= tokens; }
};

class RadixCacheIndex;

// What `node->` shows (cache_index.hpp:65-96): the node's device state when read.
struct CacheNodeView {
  uint64_t node_id = 0;
  TokenSeq edge;
  SensitivityLabel label = SensitivityLabel::PendingPrivate;
  bool private_tag = true;
  UserId creator{};
  OwnerClass owner_class = OwnerClass::Customer;
  std::vector<KvHandle> kv_handles;
  AccessStats stats;
  uint32_t span() const { return static_cast<uint32_t>(edge.size()); }
  bool is_root() const { return false; }
};

namespace b200 {
struct NodeData {
  RadixCacheIndex* index = nullptr;
  std::vector<uint64_t> h, d;  // keys of the node's whole path, root-first (one per token)
  TokenSeq path;               // its tokens
  uint32_t span = 0;           // the node's own tokens: the last `span` of the path
  uint64_t id = 0;
};
}  // namespace b200

class NodeRef {
 public:
  NodeRef() = default;
  NodeRef(std::nullptr_t) {}  // NOLINT: mirrors CacheNode* = nullptr
  explicit NodeRef(std::shared_ptr<b200::NodeData> p) : p_(std::move(p)) {}
  struct Proxy {
    CacheNodeView v;
    const CacheNodeView* operator->() const { return &v; }
  };
  Proxy operator->() const;
  explicit operator bool() const { return p_ != nullptr; }
  friend bool operator==(const NodeRef& a, std::nullptr_t) { return !a.p_; }
  friend bool operator!=(const NodeRef& a, std::nullptr_t) { return a.p_ != nullptr; }
  friend bool operator==(const NodeRef& a, const NodeRef& b) {
    if (!a.p_ || !b.p_) return a.p_ == b.p_;
    return a.p_->h.back() == b.p_->h.back() && a.p_->d.back() == b.p_->d.back() && a.p_->span == b.p_->span;
  }
  const b200::NodeData* data() const { return p_.get(); }

 private:
  std::shared_ptr<b200::NodeData> p_;
};

// cache_index.hpp:100-106
struct MatchResult {
  uint64_t matched_tokens = 0;
  std::vector<KvHandle> handles;  // covering the matched prefix, in order (one per token)
  NodeRef terminal_node = nullptr;
  MemTier lowest_tier = MemTier::HBM;
  std::vector<NodeRef> path;  // root-side first (one per matched token)
};

class RadixCacheIndex {
 public:
  struct Config {
    TierBudget budget;
    bool tiered_demotion;
    Config() : budget(TierBudget::from_tokens(1ull << 40, 0, 0)), tiered_demotion(false) {}
  };

  explicit RadixCacheIndex(Config cfg = Config(), int device = 0) : budget_(cfg.budget) {
    skv_config c;
    skv_config_default(&c);
    c.device = device;
    c.block_tokens = 1;  // token-granular, like the reference's edges
    c.window_tokens = 0;
    c.index_capacity = 1ull << 20;
    c.max_prompts = 1;
    c.max_tokens = 1ull << 16;
    c.max_window_entries = 1ull << 14;
    b200::check(skv_create(&c, &ctx_), nullptr);
    // new nodes start PendingPrivate (cache_index.hpp:196-198) until labeled
    b200::check(skv_set_label_policy(ctx_, 1), ctx_);
  }
  ~RadixCacheIndex() {
    if (ctx_) skv_destroy(ctx_);
  }
  RadixCacheIndex(const RadixCacheIndex&) = delete;
  RadixCacheIndex& operator=(const RadixCacheIndex&) = delete;

  // cache_index.hpp:152-205
  NodeRef insert(const TokenSeq& seq, UserId user, OwnerClass owner, uint64_t epoch,
                 uint32_t* new_suffix_tokens = nullptr) {
    std::lock_guard lk(mu_);
    if (seq.empty()) throw Error("insert: empty sequence");
    (void)epoch;
    auto nd = keys_of(seq);
    skv_batch b = batch_of(seq, user, owner);
    uint64_t fresh = 0;
    b200::check(skv_insert(ctx_, &b, &fresh), ctx_);
    budget_.used_tokens[0] += fresh;
    if (new_suffix_tokens) *new_suffix_tokens = static_cast<uint32_t>(fresh);
    nd->span = fresh ? static_cast<uint32_t>(fresh) : 1u;
    return make(nd);
  }

  // cache_index.hpp:213-237
  MatchResult match_prefix(const TokenSeq& seq, UserId user) {
    std::lock_guard lk(mu_);
    MatchResult m;
    if (seq.empty()) return m;
    const size_t n = seq.size();
    std::vector<uint64_t> h(n), d(n);
    std::vector<uint8_t> dec(n);
    uint32_t matched = 0;
    uint8_t tier = 0;
    skv_batch b = batch_of(seq, user, OwnerClass::Customer);
    skv_admit_out o{};
    o.block_h = h.data();
    o.block_d = d.data();
    o.decision = dec.data();
    o.matched_blocks = &matched;
    o.lowest_tier = &tier;
    b200::check(skv_lookup(ctx_, &b, &o), ctx_);
    m.matched_tokens = matched;
    m.lowest_tier = static_cast<MemTier>(tier);
    for (uint32_t i = 0; i < matched; ++i) {
      auto nd = std::make_shared<b200::NodeData>();
      nd->index = this;
      nd->h.assign(h.begin(), h.begin() + i + 1);
      nd->d.assign(d.begin(), d.begin() + i + 1);
      nd->path.assign(seq.begin(), seq.begin() + i + 1);
      nd->span = 1;
      NodeRef r = make(nd);
      m.handles.push_back(KvHandle{nd->id, m.lowest_tier, 1});
      m.path.push_back(r);
    }
    if (matched) m.terminal_node = m.path.back();
    return m;
  }

  // cache_index.hpp:296-304 (the host epoch counter of the index)
  uint64_t advance_epoch() {
    std::lock_guard lk(mu_);
    return ++epoch_;
  }
  uint64_t current_epoch() const {
    std::lock_guard lk(mu_);
    return epoch_;
  }

  // cache_index.hpp:312-315, 654-685: returns the number of nodes whose label changed (the node
  // itself, plus its descendant entries when a downgrade propagates)
  size_t set_label(NodeRef node, SensitivityLabel label, bool propagate, uint8_t audit = 0) {
    std::lock_guard lk(mu_);
    (void)audit;
    const auto* nd = data_of(node);
    return label_span(nd, nd->span, label, propagate);
  }

  // cache_index.hpp:321-343: the classification block = the last span_tokens tokens ending at
  // terminal; a private landing labels its top and everything below, a Public one every token
  size_t resolve_block(NodeRef terminal, uint32_t span_tokens, SensitivityLabel label, bool propagate,
                       uint8_t audit = 0) {
    std::lock_guard lk(mu_);
    (void)audit;
    if (span_tokens == 0) return 0;
    const auto* nd = data_of(terminal);
    if (span_tokens > nd->h.size()) throw Error("resolve_block: span exceeds path");
    return label_span(nd, span_tokens, label, propagate && is_private_class(label) &&
                                                  label != SensitivityLabel::PendingPrivate);
  }

  // cache_index.hpp:362-381: the handle's tokens move one tier down
  KvHandle demote(KvHandle handle) {
    std::lock_guard lk(mu_);
    auto it = nodes_.find(handle.id);
    if (it == nodes_.end()) throw Error("demote: unknown handle");
    auto nd = it->second.lock();
    if (!nd) throw Error("demote: stale handle");
    if (handle.tier == MemTier::SSD) throw CapacityExhausted("demote: already on the lowest tier");
    const uint8_t t = static_cast<uint8_t>(static_cast<uint8_t>(handle.tier) + 1);
    const size_t k0 = nd->h.size() - nd->span;
    std::vector<uint8_t> tiers(nd->span, t);
    const uint32_t bo[2] = {0, nd->span};
    b200::check(skv_set_tiers(ctx_, nd->h.data() + k0, nd->d.data() + k0, bo, 1, tiers.data()), ctx_);
    budget_.used_tokens[static_cast<size_t>(handle.tier)] -= std::min<uint64_t>(
        budget_.used_tokens[static_cast<size_t>(handle.tier)], nd->span);
    budget_.used_tokens[t] += nd->span;
    handle.tier = static_cast<MemTier>(t);
    return handle;
  }

  // cache_index.hpp:385-393 (the node's window lives on its first token)
  void record_access(NodeRef node, UserId user) {
    std::lock_guard lk(mu_);
    const auto* nd = data_of(node);
    const size_t k = nd->h.size() - nd->span;
    b200::check(skv_record_accesses(ctx_, &nd->h[k], &nd->d[k], &user.value, 1), ctx_);
  }
  void roll_window(NodeRef node) {
    std::lock_guard lk(mu_);
    const auto* nd = data_of(node);
    const size_t k = nd->h.size() - nd->span;
    b200::check(skv_roll_entries(ctx_, &nd->h[k], &nd->d[k], 1), ctx_);
  }

  // cache_index.hpp:422-438 (the node spelled by seq: its last token)
  NodeRef find_node(const TokenSeq& seq) {
    std::lock_guard lk(mu_);
    if (seq.empty()) return nullptr;
    auto nd = keys_of(seq);
    skv_entry e;
    uint8_t found = 0;
    b200::check(skv_get_entries(ctx_, &nd->h.back(), &nd->d.back(), 1, &e, &found), ctx_);
    if (!found) return nullptr;
    nd->span = 1;
    return make(nd);
  }

  size_t node_count() const { return static_cast<size_t>(skv_entry_count(ctx_)); }
  const TierBudget& budget() const { return budget_; }

  // the facade's device access (EntropyMonitor)
  skv_ctx* device_context() const { return ctx_; }
  std::mutex& device_mutex() const { return mu_; }
  CacheNodeView view(const b200::NodeData& nd) const {
    std::lock_guard lk(mu_);
    const size_t k0 = nd.h.size() - nd.span;
    std::vector<skv_entry> es(nd.span);
    std::vector<uint8_t> found(nd.span);
    b200::check(skv_get_entries(ctx_, nd.h.data() + k0, nd.d.data() + k0, nd.span, es.data(), found.data()), ctx_);
    CacheNodeView v;
    v.node_id = nd.id;
    v.edge.assign(nd.path.end() - nd.span, nd.path.end());
    const skv_entry& hd = es[0];
    v.label = static_cast<SensitivityLabel>(hd.label);
    v.private_tag = v.label != SensitivityLabel::Public;
    v.creator = UserId{hd.creator};
    v.owner_class = hd.owner ? OwnerClass::Business : OwnerClass::Customer;
    uint8_t tier = 0;
    for (const auto& e : es) tier = std::max(tier, e.tier);
    v.kv_handles.push_back(KvHandle{nd.id, static_cast<MemTier>(tier), nd.span});
    v.stats.hit_cur = hd.hit_cur;
    v.stats.u_cnt = hd.u_cnt;
    v.stats.hit_pre = hd.hit_pre;
    v.stats.u_pre = hd.u_pre;
    return v;
  }
  // a node named by one entry key (monitor events)
  NodeRef node_of_key(uint64_t h, uint64_t d) {
    std::lock_guard lk(mu_);
    auto nd = std::make_shared<b200::NodeData>();
    nd->index = this;
    nd->h = {h};
    nd->d = {d};
    nd->path = {0};
    nd->span = 1;
    return make(nd);
  }

 private:
  static const b200::NodeData* data_of(const NodeRef& n) {
    if (!n.data()) throw Error("null NodeRef");
    return n.data();
  }
  skv_batch batch_of(const TokenSeq& seq, UserId user, OwnerClass owner) {
    off_[0] = 0;
    off_[1] = seq.size();
    user_ = user.value;
    owner_ = owner == OwnerClass::Business ? 1 : 0;
    skv_batch b{};
    b.tokens = seq.data();
    b.offsets = off_;
    b.users = &user_;
    b.owners = &owner_;
    b.n_prompts = 1;
    b.n_tokens = seq.size();
    b.on_device = 0;
    return b;
  }
  std::shared_ptr<b200::NodeData> keys_of(const TokenSeq& seq) {
    auto nd = std::make_shared<b200::NodeData>();
    nd->index = this;
    nd->path = seq;
    nd->h.resize(seq.size());
    nd->d.resize(seq.size());
    skv_batch b = batch_of(seq, UserId{0}, OwnerClass::Customer);
    skv_admit_out o{};
    o.block_h = nd->h.data();
    o.block_d = nd->d.data();
    b200::check(skv_lookup(ctx_, &b, &o), ctx_);
    return nd;
  }
  NodeRef make(std::shared_ptr<b200::NodeData> nd) {
    nd->id = ++next_id_;
    nodes_[nd->id] = nd;
    return NodeRef(std::move(nd));
  }
  size_t label_span(const b200::NodeData* nd, uint32_t span, SensitivityLabel label, bool propagate) {
    const size_t k0 = nd->h.size() - span;
    std::vector<skv_entry> es(span);
    std::vector<uint8_t> found(span);
    b200::check(skv_get_entries(ctx_, nd->h.data() + k0, nd->d.data() + k0, span, es.data(), found.data()), ctx_);
    for (uint8_t f : found)
      if (!f) throw Error("set_label: node not in the index");
    if (es[0].label == static_cast<uint8_t>(SensitivityLabel::Public) && label == SensitivityLabel::PendingPrivate)
      throw IllegalTransition("Public -> PendingPrivate is not allowed");
    size_t own = 0;
    for (const auto& e : es) own += e.label != static_cast<uint8_t>(label);
    size_t changed = 0;
    b200::check(skv_label_entries(ctx_, nd->h.data() + k0, nd->d.data() + k0, span, static_cast<uint8_t>(label),
                                  propagate ? 1 : 0, &changed),
                ctx_);
    return (own ? 1 : 0) + (changed - own);
  }

  skv_ctx* ctx_ = nullptr;
  mutable std::mutex mu_;
  TierBudget budget_;
  uint64_t epoch_ = 0;
  uint64_t next_id_ = 0;
  std::map<uint64_t, std::weak_ptr<b200::NodeData>> nodes_;
  uint64_t off_[2] = {0, 0};
  uint64_t user_ = 0;
  uint8_t owner_ = 0;
};

inline NodeRef::Proxy NodeRef::operator->() const {
  if (!p_) throw Error("null NodeRef");
  return Proxy{p_->index->view(*p_)};
}

namespace b200 {
inline skv_ctx* util_ctx() {
  static std::unique_ptr<RadixCacheIndex> holder = std::make_unique<RadixCacheIndex>();
  return holder->device_context();
}
}  // namespace b200

}  // namespace safekv
