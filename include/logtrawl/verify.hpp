#pragma once
// Drop-in for logtrawl/verify.hpp (reference: /root/reference/proj/include/
// logtrawl/verify.hpp).  verify_hits runs the stage-2 suffix compare and the
// order-preserving compaction on the B200; Alert names and line numbers are
// attached on the host (LineIndex stays a host index, as in the reference).
#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

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

struct DeviceRules {
  glop_rules* r = nullptr;
  explicit DeviceRules(const RuleSet& rules, std::size_t prefix_len) {
    std::string blob;
    std::vector<std::uint64_t> off{0};
    for (std::size_t i = 0; i < rules.patterns.size(); ++i) {
      if (rules.patterns[i].id != i) throw std::invalid_argument("verify_hits: pattern ids must be dense 0..k-1");
      blob += rules.patterns[i].bytes;
      off.push_back(blob.size());
    }
    check(glop_rules_upload(context(), reinterpret_cast<const std::uint8_t*>(blob.data()), off.data(),
                            static_cast<std::uint32_t>(rules.patterns.size()), prefix_len, &r),
          "verify_hits");
  }
  ~DeviceRules() { glop_rules_destroy(r); }
  DeviceRules(const DeviceRules&) = delete;
  DeviceRules& operator=(const DeviceRules&) = delete;
};

}  // namespace detail

// verify.hpp:69-105 on the B200: alerts sorted by (offset, rule_id).
inline std::vector<Alert> verify_hits(std::string_view text, const std::vector<Hit>& hits, const PrefixSet& prefixes,
                                      const RuleSet& rules, const LineIndex* lines = nullptr) {
  std::vector<Alert> out;
  if (hits.empty()) return out;
  detail::DeviceRules dr(rules, prefixes.prefix_len);
  glop_alert* a = nullptr;
  std::uint64_t na = 0;
  detail::check(glop_verify_hits(detail::context(), dr.r, reinterpret_cast<const std::uint8_t*>(text.data()),
                                 text.size(), 0, reinterpret_cast<const glop_hit*>(hits.data()), hits.size(), 0, &a,
                                 &na, nullptr),
                "verify_hits");
  out.reserve(na);
  for (std::uint64_t i = 0; i < na; ++i) {
    Alert al;
    al.offset = a[i].offset;
    al.line = lines ? lines->line_of(a[i].offset) : 0;
    al.rule_id = a[i].rule_id;
    al.rule_name = rules.patterns[a[i].rule_id].name;
    al.pattern_len = a[i].pattern_len;
    al.verified = true;
    out.push_back(std::move(al));
  }
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
