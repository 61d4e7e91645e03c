#pragma once
// Drop-in for logtrawl/scan.hpp (reference: /root/reference/proj/include/
// logtrawl/scan.hpp).  pfac_scan keeps its signature and result (every start
// position walks the failureless trie; a Hit per output of every visited
// state; sorted by (offset, pattern_id)) but runs on the B200 through the C
// ABI.  ScanConfig::workers is accepted and ignored: results never depend on
// it, and the device decides its own parallelism.
#include <cstdint>
#include <cstring>
#include <string_view>
#include <thread>
#include <vector>

#include "glop.h"
#include "logtrawl/automaton.hpp"
#include "logtrawl/detail/abi.hpp"
#include "logtrawl/rules.hpp"

namespace logtrawl {

struct Hit {  // scan.hpp:31-41; layout-identical to glop_hit
  std::size_t offset = 0;
  std::uint32_t pattern_id = 0;
  std::uint32_t matched_len = 0;

  friend bool operator==(const Hit&, const Hit&) = default;
  friend bool operator<(const Hit& x, const Hit& y) {
    return x.offset < y.offset || (x.offset == y.offset && x.pattern_id < y.pattern_id);
  }
};
static_assert(sizeof(Hit) == sizeof(glop_hit), "Hit must stay layout-identical to glop_hit");

struct ScanConfig {  // scan.hpp:43-47
  unsigned workers = 1;
  std::size_t chunk_size = 0;
  std::size_t overlap = 0;
};

inline unsigned default_workers() {  // scan.hpp:49-52
  const unsigned hw = std::thread::hardware_concurrency();
  return hw ? hw : 1;
}

namespace detail {

// Device copy of `a`, uploaded once and reused while the value's buffers are
// unchanged.  Compact automata are re-expanded to the dense goto table the
// ABI consumes.
inline glop_trie* device_trie(const Automaton& a) {
  std::shared_ptr<DeviceTrieCache> cache = a.device;
  if (!cache) a.device = cache = std::make_shared<DeviceTrieCache>();
  const void* key[4] = {a.dense_table.data(), a.cnodes.data(), a.packed.data(), a.out_flat.data()};
  const std::size_t sizes[3] = {a.state_count, a.dense_table.size() + a.packed.size(), a.out_flat.size()};
  std::lock_guard<std::mutex> lk(cache->mu);
  if (cache->trie && std::memcmp(cache->key, key, sizeof key) == 0 &&
      std::memcmp(cache->sizes, sizes, sizeof sizes) == 0)
    return cache->trie;
  if (cache->trie) {  // a copy with different buffers: give it its own cache
    auto fresh = std::make_shared<DeviceTrieCache>();
    a.device = fresh;
    return device_trie(a);
  }
  std::vector<std::int32_t> dense_local;
  const std::int32_t* dense = a.dense_table.data();
  if (a.backend == Backend::compact) {
    dense_local.assign(a.state_count * 256, kNoTransition);
    for (std::size_t s = 0; s < a.state_count; ++s)
      for (unsigned b = 0; b < 256; ++b)
        dense_local[s * 256 + b] = a.goto_edge(static_cast<std::int32_t>(s), static_cast<unsigned char>(b));
    dense = dense_local.data();
  }
  glop_trie* t = nullptr;
  check(glop_trie_upload(context(), dense, static_cast<std::uint32_t>(a.state_count), a.out_offsets.data(),
                         reinterpret_cast<const glop_output*>(a.out_flat.data()), &t),
        "pfac_scan");
  cache->trie = t;
  std::memcpy(cache->key, key, sizeof key);
  std::memcpy(cache->sizes, sizes, sizeof sizes);
  return t;
}

}  // namespace detail

// scan.hpp:177-202 on the B200.
inline std::vector<Hit> pfac_scan(std::string_view text, const Automaton& a, const ScanConfig& cfg = {}) {
  (void)cfg;
  if (a.kind != AutomatonKind::failureless) throw std::invalid_argument("pfac_scan: automaton must be failureless");
  std::vector<Hit> hits;
  if (text.empty()) return hits;
  glop_trie* t = detail::device_trie(a);
  glop_hit* h = nullptr;
  std::uint64_t nh = 0;
  detail::check(glop_pfac_scan(detail::context(), t, reinterpret_cast<const std::uint8_t*>(text.data()),
                               text.size(), 0, &h, &nh),
                "pfac_scan");
  hits.resize(nh);
  if (nh) std::memcpy(hits.data(), h, nh * sizeof(Hit));
  glop_free(h);
  return hits;
}

// Every occurrence of every full pattern, sorted (scan.hpp:247-260).  Served
// by the device PFAC path with untruncated prefixes (L = max_len), which
// reports exactly the full-pattern occurrences.
inline std::vector<Match> naive_scan(std::string_view text, const RuleSet& rules) {
  std::vector<Match> out;
  if (text.empty() || rules.patterns.empty()) return out;
  const Automaton trie = build_failureless_trie(truncate_prefixes(rules, std::max<std::size_t>(rules.max_len, 1)));
  for (const Hit& h : pfac_scan(text, trie)) out.push_back(Match{h.offset, h.pattern_id});
  return out;
}

}  // namespace logtrawl
