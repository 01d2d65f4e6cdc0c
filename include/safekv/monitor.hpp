// monitor.hpp -- drop-in facade of the reference's EntropyMonitor (proj/include/safekv/
// monitor.hpp:12-113) over the device monitor: check_anomaly and epoch_pass evaluate the FP64
// suspicion predicate and relabel on the device (skv_check_anomaly / skv_epoch).
#pragma once

#include <functional>
#include <utility>
#include <vector>

#include "access_stats.hpp"
#include "cache_index.hpp"
#include "core.hpp"

namespace safekv {

struct MonitorConfig {
  double entropy_jump = 0.3;
  uint64_t u_pre_max = 1;
};

enum class AnomalyAction : uint8_t { None = 0, DowngradeToPrivate = 1, Restrict = 2 };

inline const char* to_string(AnomalyAction a) {
  switch (a) {
    case AnomalyAction::DowngradeToPrivate: return "downgrade_to_private";
    case AnomalyAction::Restrict: return "restrict";
    default: return "none";
  }
}

struct AnomalyEvent {
  NodeRef node = nullptr;
  uint64_t node_id = 0;
  double entropy_now = 0.0;
  double entropy_prev = 0.0;
  uint64_t u_pre = 0;
  AnomalyAction action = AnomalyAction::None;
  uint64_t epoch = 0;
  OwnerClass owner_class = OwnerClass::Customer;
};

class EntropyMonitor {
 public:
  EntropyMonitor(RadixCacheIndex& index, MonitorConfig cfg = {}) : index_(index), cfg_(cfg) {
    std::lock_guard lk(index_.device_mutex());
    b200::check(skv_set_monitor_config(index_.device_context(), cfg.entropy_jump, cfg.u_pre_max),
                index_.device_context());
  }

  void set_alert_sink(std::function<void(const AnomalyEvent&)> sink) { sink_ = std::move(sink); }

  void record_access(NodeRef node, UserId user) { index_.record_access(node, user); }

  // monitor.hpp:56-81 (on the node's window: its first token's entry)
  AnomalyEvent check_anomaly(NodeRef node, uint64_t epoch) {
    const auto* nd = node.data();
    if (!nd) throw Error("null NodeRef");
    const size_t k = nd->h.size() - nd->span;
    skv_event ev{};
    int fired = 0;
    {
      std::lock_guard lk(index_.device_mutex());
      b200::check(skv_check_anomaly(index_.device_context(), nd->h[k], nd->d[k], epoch, &ev, &fired),
                  index_.device_context());
    }
    AnomalyEvent out = from_device(ev, node, epoch);
    if (!fired) out.action = AnomalyAction::None;
    if (out.action != AnomalyAction::None) emit(out);
    return out;
  }

  // monitor.hpp:85-99: every Public entry with window activity checked (ancestors first, a fired
  // entry relabeling its subtree), then every window rolled -- one device pass
  std::vector<AnomalyEvent> epoch_pass(uint64_t epoch) {
    std::vector<skv_event> evs(256);
    size_t n = 0;
    uint64_t dev_epoch = 0;
    {
      std::lock_guard lk(index_.device_mutex());
      skv_ctx* c = index_.device_context();
      b200::check(skv_epoch(c, evs.data(), evs.size(), &n, &dev_epoch), c);
      if (n > evs.size()) {
        evs.resize(n);
        b200::check(skv_last_events(c, evs.data(), n, &n), c);
      }
    }
    std::vector<AnomalyEvent> fired;
    for (size_t i = 0; i < n; ++i) {
      AnomalyEvent e = from_device(evs[i], index_.node_of_key(evs[i].h, evs[i].d), epoch);
      emit(e);
      fired.push_back(e);
    }
    alerts_last_epoch_ = fired.size();
    total_alerts_ += fired.size();
    return fired;
  }

  uint64_t alerts_last_epoch() const { return alerts_last_epoch_; }
  uint64_t total_alerts() const { return total_alerts_; }

 private:
  static AnomalyEvent from_device(const skv_event& ev, NodeRef node, uint64_t epoch) {
    AnomalyEvent e;
    e.node = node;
    e.node_id = node.data() ? node.data()->id : 0;
    e.entropy_now = ev.entropy_now;
    e.entropy_prev = ev.entropy_prev;
    e.u_pre = ev.u_pre;
    e.action = static_cast<AnomalyAction>(ev.action);
    e.epoch = epoch;
    e.owner_class = ev.owner ? OwnerClass::Business : OwnerClass::Customer;
    return e;
  }
  void emit(const AnomalyEvent& ev) {
    if (sink_) sink_(ev);
  }

  RadixCacheIndex& index_;
  MonitorConfig cfg_;
  std::function<void(const AnomalyEvent&)> sink_;
  uint64_t alerts_last_epoch_ = 0;
  uint64_t total_alerts_ = 0;
};

}  // namespace safekv
