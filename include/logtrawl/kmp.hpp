#pragma once
// Drop-in for logtrawl/kmp.hpp (reference: /root/reference/proj/include/
// logtrawl/kmp.hpp).  The failure table stays a host computation; the search
// runs on the B200 as a chunk-parallel KMP with an (m-1)-byte warm-up overlap
// per chunk, reporting the same ascending, overlapping offsets and exactly the
// sequential algorithm's comparison count.  A failure table that is not the
// pattern's prefix function (the reference runs whatever table it is given),
// or a pattern of 8,192 bytes or more, runs the reference's sequential loop on
// one device thread instead -- same results, no parallelism.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string_view>
#include <vector>

#include "glop.h"
#include "logtrawl/detail/abi.hpp"
#include "logtrawl/rules.hpp"

namespace logtrawl {

struct FailureTable {  // kmp.hpp:20-23
  std::uint32_t pattern_id = 0;
  std::vector<std::uint32_t> table;
};

// Prefix function: table[i] = longest proper border of pattern[0..=i]
// (kmp.hpp:25-36).
inline FailureTable build_failure_table(const Pattern& p) {
  FailureTable ft;
  ft.pattern_id = p.id;
  const std::size_t m = p.bytes.size();
  ft.table.assign(m, 0);
  std::uint32_t border = 0;
  for (std::size_t i = 1; i < m; ++i) {
    while (border && p.bytes[i] != p.bytes[border]) border = ft.table[border - 1];
    if (p.bytes[i] == p.bytes[border]) ++border;
    ft.table[i] = border;
  }
  return ft;
}

// kmp.hpp:41-69 on the B200.
inline std::vector<std::size_t> kmp_search(std::string_view text, const Pattern& p, const FailureTable& ft,
                                           std::uint64_t* comparisons = nullptr) {
  std::vector<std::size_t> out;
  const std::size_t m = p.bytes.size();
  if (m == 0 || text.size() < m) return out;
  if (ft.table.size() != m) throw std::invalid_argument("kmp_search: failure table does not match pattern");
  std::uint64_t* offs = nullptr;
  std::uint64_t no = 0;
  detail::check(glop_group_kmp_search(detail::group(), reinterpret_cast<const std::uint8_t*>(p.bytes.data()),
                                      static_cast<std::uint32_t>(m), ft.table.data(),
                                      reinterpret_cast<const std::uint8_t*>(text.data()), text.size(), &offs, &no,
                                      comparisons),
                "kmp_search");
  out.assign(offs, offs + no);
  glop_free(offs);
  return out;
}

// One device pass per pattern, merged by (offset, pattern_id) (kmp.hpp:74-94).
inline std::vector<Match> kmp_multi(std::string_view text, const RuleSet& rules,
                                    const std::vector<FailureTable>* prebuilt = nullptr,
                                    std::uint64_t* comparisons = nullptr) {
  std::vector<Match> out;
  for (const Pattern& p : rules.patterns) {
    const FailureTable local = prebuilt ? FailureTable{} : build_failure_table(p);
    const FailureTable& ft = prebuilt ? (*prebuilt)[p.id] : local;
    for (const std::size_t off : kmp_search(text, p, ft, comparisons)) out.push_back(Match{off, p.id});
  }
  std::sort(out.begin(), out.end());
  return out;
}

}  // namespace logtrawl
