#pragma once
// Drop-in for logtrawl/verify.hpp (reference: /root/reference/proj/include/
// logtrawl/verify.hpp).  verify_hits runs the stage-2 suffix compare and the
// order-preserving compaction on the B200; Alert names are attached on the
// host.  LineIndex stays the reference's host index; run_engine_scan computes
// the alert lines on the device from the same upload (pipeline.hpp).
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include <sys/mman.h>

#include "glop.h"
#include "logtrawl/detail/abi.hpp"
#include "logtrawl/rules.hpp"
#include "logtrawl/scan.hpp"

namespace logtrawl {

struct Alert {  // verify.hpp:19-28
  std::size_t offset = 0;
  std::size_t line = 0;
  std::uint32_t rule_id = 0;
  std::string rule_name;
  std::uint32_t pattern_len = 0;
  bool verified = false;
  friend bool operator==(const Alert&, const Alert&) = default;
};

struct ScanReport {  // verify.hpp:30-36
  std::vector<Alert> alerts;
  std::size_t total_matches = 0;
  std::size_t stage1_hits = 0;
  std::size_t stage1_rejected = 0;
  std::size_t bytes_scanned = 0;
};

// Offset -> 1-based line; an LF belongs to the line it ends (verify.hpp:40-64).
class LineIndex {
 public:
  explicit LineIndex(std::string_view text) {
    starts_.push_back(0);
    if (text.empty()) return;
    const char* base = text.data();
    for (const char* p = base; (p = static_cast<const char*>(std::memchr(p, '\n', text.size() - (p - base))));) {
      ++p;
      starts_.push_back(static_cast<std::size_t>(p - base));
      if (static_cast<std::size_t>(p - base) >= text.size()) break;
    }
  }
  std::size_t line_of(std::size_t offset) const {
    return static_cast<std::size_t>(std::upper_bound(starts_.begin(), starts_.end(), offset) - starts_.begin());
  }
  std::size_t line_begin(std::size_t line) const { return starts_.at(line - 1); }
  std::size_t line_count() const { return starts_.size(); }

 private:
  std::vector<std::size_t> starts_;
};

namespace detail {

// Device alerts -> reference Alerts.  The device reports the POSITION of the
// pattern (hits name patterns by position: rules.patterns.at(pattern_id),
// verify.hpp:78); the Alert carries that pattern's id and name, sorted by
// (offset, rule_id) (verify.hpp:100-103) -- only a RuleSet whose ids are not
// their positions changes the device's (offset, position) order.
// n default Alerts, the storage backed by huge pages where the kernel allows
// it (2M alerts are 128 MB: 4 KB first-touch faults were most of the cost).
inline std::vector<Alert> alert_storage(std::size_t n) {
  std::vector<Alert> v;
  v.reserve(n);
#ifdef MADV_HUGEPAGE
  const std::uintptr_t huge = std::uintptr_t(2) << 20;
  const std::uintptr_t lo = (reinterpret_cast<std::uintptr_t>(v.data()) + huge - 1) & ~(huge - 1);
  const std::uintptr_t hi = reinterpret_cast<std::uintptr_t>(v.data() + n) & ~(huge - 1);
  if (hi > lo) (void)madvise(reinterpret_cast<void*>(lo), hi - lo, MADV_HUGEPAGE);
#endif
  v.resize(n);
  return v;
}

// glop_alert records -> Alerts (the reference's Alert values).  `storage`:
// default Alerts prepared while the device worked (any size; resized here).
inline std::vector<Alert> to_alerts(const glop_alert* a, std::uint64_t na, const RuleSet& rules,
                                    const LineIndex* lines, const std::uint64_t* dev_lines,
                                    std::vector<Alert> storage = {}) {
  for (std::uint64_t i = 0; i < na; ++i)  // rules.patterns.at() (verify.hpp:78) throws before any work
    if (a[i].rule_id >= rules.patterns.size()) (void)rules.patterns.at(a[i].rule_id);
  std::vector<Alert> out = storage.capacity() >= na ? std::move(storage) : alert_storage(na);
  out.resize(na);
  std::atomic<bool> dense_ids{true};
  parallel_for(na, [&](std::size_t lo, std::size_t hi) {
    bool dense = true;
    for (std::size_t i = lo; i < hi; ++i) {
      const Pattern& p = rules.patterns[a[i].rule_id];
      dense = dense && p.id == a[i].rule_id;
      Alert& al = out[i];
      al.offset = a[i].offset;
      al.line = dev_lines ? dev_lines[i] : (lines ? lines->line_of(a[i].offset) : 0);
      al.rule_id = p.id;
      al.rule_name = p.name;
      al.pattern_len = a[i].pattern_len;
      al.verified = true;
    }
    if (!dense) dense_ids = false;
  });
  if (!dense_ids)
    std::stable_sort(out.begin(), out.end(), [](const Alert& x, const Alert& y) {
      return x.offset != y.offset ? x.offset < y.offset : x.rule_id < y.rule_id;
    });
  return out;
}

}  // namespace detail

// verify.hpp:69-105 on the B200: alerts sorted by (offset, rule_id).  The
// rule set's device copy is cached by content (detail::device_rules).
inline std::vector<Alert> verify_hits(std::string_view text, const std::vector<Hit>& hits, const PrefixSet& prefixes,
                                      const RuleSet& rules, const LineIndex* lines = nullptr) {
  if (hits.empty()) return {};
  const auto dr = detail::device_rules(rules, prefixes.prefix_len);
  glop_alert* a = nullptr;
  std::uint64_t na = 0;
  detail::check(glop_verify_hits(detail::context(), glop_group_rules_member(dr->rules, 0),
                                 reinterpret_cast<const std::uint8_t*>(text.data()),
                                 text.size(), 0, reinterpret_cast<const glop_hit*>(hits.data()), hits.size(), 0, &a,
                                 &na, nullptr),
                "verify_hits");
  std::vector<Alert> out = detail::to_alerts(a, na, rules, lines, nullptr);
  glop_free(a);
  return out;
}

inline ScanReport assemble_report(std::vector<Alert> alerts, std::size_t stage1_hits,
                                  std::size_t bytes_scanned) {  // verify.hpp:107-117
  ScanReport r;
  r.total_matches = alerts.size();
  r.stage1_hits = stage1_hits;
  r.stage1_rejected = stage1_hits - r.total_matches;
  r.bytes_scanned = bytes_scanned;
  r.alerts = std::move(alerts);
  return r;
}

}  // namespace logtrawl
