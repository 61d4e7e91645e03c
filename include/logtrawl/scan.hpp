#pragma once
// Drop-in for logtrawl/scan.hpp (reference: /root/reference/proj/include/
// logtrawl/scan.hpp).  pfac_scan keeps its signature and result (every start
// position walks the failureless trie; a Hit per output of every visited
// state; sorted by (offset, pattern_id)) but runs on the B200s of the process
// group (detail::group(): every visible GPU, or GLOP_DEVICES) through the C
// ABI.  ScanConfig::workers is accepted and ignored: results never depend on
// it, and the devices decide their own parallelism.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
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

// The automaton's device-copy slot.  Copies of an Automaton share it until
// one of them is found to hold different buffers; reads and replacements of
// the slot are serialised here (concurrent first scans of one value race for
// nothing).  An Automaton must not be mutated in place after its first scan:
// the slot is keyed on its buffers' addresses and sizes, not their contents.
inline std::mutex& slot_mutex() {
  static std::mutex mu;
  return mu;
}
inline std::shared_ptr<DeviceTrieCache> cache_slot(const Automaton& a, bool fresh = false) {
  std::lock_guard<std::mutex> lk(slot_mutex());
  if (!a.device || fresh) a.device = std::make_shared<DeviceTrieCache>();
  return a.device;
}

// Uploads (dense goto table, CSR outputs) once per automaton value.
template <typename Build>
inline glop_group_trie* cached_trie(const Automaton& a, const char* what, Build&& build) {
  std::shared_ptr<DeviceTrieCache> cache = cache_slot(a);
  const void* key[4] = {a.dense_table.data(), a.cnodes.data(), a.packed.data(), a.out_flat.data()};
  const std::size_t sizes[3] = {a.state_count, a.dense_table.size() + a.packed.size(), a.out_flat.size()};
  for (int attempt = 0; attempt < 2; ++attempt) {
    std::lock_guard<std::mutex> lk(cache->mu);
    if (cache->trie && std::memcmp(cache->key, key, sizeof key) == 0 &&
        std::memcmp(cache->sizes, sizes, sizeof sizes) == 0)
      return cache->trie;
    if (!cache->trie) {
      cache->trie = build(what);
      std::memcpy(cache->key, key, sizeof key);
      std::memcpy(cache->sizes, sizes, sizeof sizes);
      return cache->trie;
    }
    // a copy with different buffers: give this value its own slot
    cache = cache_slot(a, true);
  }
  throw std::logic_error("glop: device trie cache");
}

// The reference's dense goto table (compact automata are re-expanded).
inline std::vector<std::int32_t> dense_goto(const Automaton& a) {
  if (a.backend == Backend::dense) return a.dense_table;
  std::vector<std::int32_t> dense(a.state_count * 256, kNoTransition);
  for (std::size_t s = 0; s < a.state_count; ++s)
    for (unsigned b = 0; b < 256; ++b)
      dense[s * 256 + b] = a.goto_edge(static_cast<std::int32_t>(s), static_cast<unsigned char>(b));
  return dense;
}

// Device copies (one per group device) of a failureless trie (pfac_scan).
inline glop_group_trie* device_trie(const Automaton& a) {
  return cached_trie(a, "pfac_scan", [&](const char* what) {
    const std::vector<std::int32_t> dense = dense_goto(a);
    glop_group_trie* t = nullptr;
    check(glop_group_trie_upload(group(), dense.data(), static_cast<std::uint32_t>(a.state_count),
                                 a.out_offsets.data(), reinterpret_cast<const glop_output*>(a.out_flat.data()), &t),
          what);
    return t;
  });
}

// Device copy of a full Aho-Corasick automaton for chunked_ac_scan: its goto
// trie (the dense table holds raw goto edges, automaton.hpp:57) with only each
// pattern's own output (matched_len == depth; the failure-merged outputs are
// what the device's per-start walk finds by itself).
inline glop_group_trie* device_ac_trie(const Automaton& a) {
  return cached_trie(a, "chunked_ac_scan", [&](const char* what) {
    const std::vector<std::int32_t> dense = dense_goto(a);
    std::vector<std::uint32_t> off(a.state_count + 1, 0);
    std::vector<AutomatonOutput> flat;
    for (std::size_t s = 0; s < a.state_count; ++s) {
      off[s] = static_cast<std::uint32_t>(flat.size());
      for (const AutomatonOutput& o : a.outputs[s])
        if (o.matched_len == a.depth[s] && o.matched_len > 0) flat.push_back(o);
    }
    off[a.state_count] = static_cast<std::uint32_t>(flat.size());
    glop_group_trie* t = nullptr;
    check(glop_group_trie_upload(group(), dense.data(), static_cast<std::uint32_t>(a.state_count), off.data(),
                                 reinterpret_cast<const glop_output*>(flat.data()), &t),
          what);
    return t;
  });
}

}  // namespace detail

// scan.hpp:177-202 on the B200.
inline std::vector<Hit> pfac_scan(std::string_view text, const Automaton& a, const ScanConfig& cfg = {}) {
  (void)cfg;
  if (a.kind != AutomatonKind::failureless) throw std::invalid_argument("pfac_scan: automaton must be failureless");
  std::vector<Hit> hits;
  if (text.empty()) return hits;
  glop_group_trie* t = detail::device_trie(a);
  glop_hit* h = nullptr;
  std::uint64_t nh = 0;
  detail::check(glop_group_pfac_scan(detail::group(), t, reinterpret_cast<const std::uint8_t*>(text.data()),
                                     text.size(), &h, &nh),
                "pfac_scan");
  hits.resize(nh);
  if (nh) std::memcpy(hits.data(), h, nh * sizeof(Hit));
  glop_free(h);
  return hits;
}

// scan.hpp:207-243 on the B200: chunk k owns starts [k*c, (k+1)*c) and is
// walked from the root over [k*c, min(k*c + c + overlap, n)); a match is
// reported only when its chunk owns its start and reaches its end, so an
// overlap below max_len - 1 loses straddling matches exactly as the reference
// does.  cfg.workers is ignored (results never depend on it).
inline std::vector<Match> chunked_ac_scan(std::string_view text, const Automaton& a, const ScanConfig& cfg) {
  if (a.kind != AutomatonKind::full_ac) throw std::invalid_argument("chunked_ac_scan: automaton must be full_ac");
  std::vector<Match> out;
  const std::size_t n = text.size();
  if (n == 0) return out;
  glop_trie* t = glop_group_trie_member(detail::device_ac_trie(a), 0);
  glop_hit* h = nullptr;
  std::uint64_t nh = 0;
  detail::check(glop_chunked_ac_scan(detail::context(), t, reinterpret_cast<const std::uint8_t*>(text.data()), n, 0,
                                     cfg.chunk_size, cfg.overlap, &h, &nh),
                "chunked_ac_scan");
  out.reserve(nh);
  for (std::uint64_t i = 0; i < nh; ++i) out.push_back(Match{h[i].offset, h[i].pattern_id});
  glop_free(h);
  // an empty pattern sits on the root: the reference's walk reports it after
  // every byte it reads, at start j + 1 when the chunk owns that start
  bool empty_pattern = false;
  std::vector<std::uint32_t> empty_ids;
  if (!a.outputs.empty())
    for (const AutomatonOutput& o : a.outputs[0])
      if (o.matched_len == 0) empty_ids.push_back(o.pattern_id), empty_pattern = true;
  if (empty_pattern) {
    const std::size_t c = cfg.chunk_size ? cfg.chunk_size : n;
    for (std::size_t k0 = 0; k0 < n; k0 += c) {
      const std::size_t own_end = std::min(k0 + c, n), scan_end = std::min(k0 + c + cfg.overlap, n);
      for (std::size_t j = k0; j < scan_end && j + 1 < own_end; ++j)
        for (std::uint32_t id : empty_ids) out.push_back(Match{j + 1, id});
    }
    std::sort(out.begin(), out.end());
  }
  return out;
}

// Brute-force ground truth (scan.hpp:245-260): a direct byte comparison of
// every pattern at every position, on the host -- the oracle engine
// equivalences are tested against, so it never runs on the device.
inline std::vector<Match> naive_scan(std::string_view text, const RuleSet& rules) {
  std::vector<Match> matches;
  for (const Pattern& p : rules.patterns) {
    const std::size_t m = p.bytes.size();
    if (m == 0 || text.size() < m) continue;
    for (std::size_t i = 0; i + m <= text.size(); ++i)
      if (std::memcmp(text.data() + i, p.bytes.data(), m) == 0) matches.push_back({i, p.id});
  }
  std::sort(matches.begin(), matches.end());
  return matches;
}

}  // namespace logtrawl
