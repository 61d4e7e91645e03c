#pragma once
// Drop-in for logtrawl/jsonl.hpp (reference: /root/reference/proj/include/
// logtrawl/jsonl.hpp:14-34): one JSON object per alert, then one summary
// object.  Field names are the reference's stability contract; the bytes
// match nlohmann::json::dump() of the reference (object keys in sorted
// order, compact separators, the same string escapes) without depending on
// the vendored json.hpp.
#include <cstdio>
#include <string>
#include <string_view>

#include "logtrawl/verify.hpp"

namespace logtrawl {

namespace detail {

inline void json_string(std::string& out, std::string_view s) {
  out += '"';
  for (unsigned char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      default:
        if (c < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof buf, "\\u%04x", c);
          out += buf;
        } else {
          out += static_cast<char>(c);
        }
    }
  }
  out += '"';
}

inline void json_field(std::string& out, const char* key, std::size_t v, bool first = false) {
  if (!first) out += ',';
  json_string(out, key);
  out += ':';
  out += std::to_string(v);
}

}  // namespace detail

inline std::string render_alerts_jsonl(const std::string& file, const ScanReport& report) {
  std::string out;
  for (const Alert& a : report.alerts) {  // keys sorted: file line offset rule rule_id
    out += '{';
    detail::json_string(out, "file");
    out += ':';
    detail::json_string(out, file);
    detail::json_field(out, "line", a.line);
    detail::json_field(out, "offset", a.offset);
    out += ',';
    detail::json_string(out, "rule");
    out += ':';
    detail::json_string(out, a.rule_name);
    detail::json_field(out, "rule_id", a.rule_id);
    out += "}\n";
  }
  out += '{';  // bytes_scanned file stage1_hits stage1_rejected total_matches
  detail::json_field(out, "bytes_scanned", report.bytes_scanned, true);
  out += ',';
  detail::json_string(out, "file");
  out += ':';
  detail::json_string(out, file);
  detail::json_field(out, "stage1_hits", report.stage1_hits);
  detail::json_field(out, "stage1_rejected", report.stage1_rejected);
  detail::json_field(out, "total_matches", report.total_matches);
  out += "}\n";
  return out;
}

}  // namespace logtrawl
