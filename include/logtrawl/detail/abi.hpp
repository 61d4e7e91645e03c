#pragma once
// Glue between the drop-in C++ API and the C ABI (include/glop.h): one
// process-wide context per device and the mapping of glop_status codes onto
// the exception types the reference throws.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <vector>
#include <new>
#include <stdexcept>
#include <string>
#include <thread>

#include "glop.h"
#include "logtrawl/automaton.hpp"
#include "logtrawl/rules.hpp"

namespace logtrawl::detail {

// GLOP_DEVICE selects the CUDA device (default 0).
inline glop_ctx* context() {
  static std::once_flag once;
  static glop_ctx* ctx = nullptr;
  static glop_status st = GLOP_OK;
  static std::string err;
  std::call_once(once, [] {
    const char* env = std::getenv("GLOP_DEVICE");
    st = glop_ctx_create(env ? std::atoi(env) : 0, &ctx);
    if (st != GLOP_OK) err = glop_last_error();
  });
  if (st != GLOP_OK) throw std::runtime_error("glop: no usable B200 device: " + err);
  return ctx;
}

// Rethrows a failed ABI call as the reference's exception type.
inline void check(glop_status s, const char* what) {
  if (s == GLOP_OK) return;
  const std::string msg = std::string(what) + ": " + glop_last_error();
  switch (s) {
    case GLOP_EINVAL: throw std::invalid_argument(msg);
    case GLOP_ELOGIC: throw std::logic_error(msg);
    case GLOP_ENOMEM: throw std::bad_alloc();
    default: throw std::runtime_error(msg);
  }
}

// fn(begin, end) over [0, n) on up to hardware_concurrency host threads
// (host-side result assembly: millions of Alert records per scan).
template <typename Fn>
inline void parallel_for(std::size_t n, Fn&& fn, std::size_t grain = 1 << 16) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const std::size_t T = std::min<std::size_t>(hw, (n + grain - 1) / grain);
  if (T <= 1) {
    if (n) fn(std::size_t{0}, n);
    return;
  }
  std::vector<std::thread> pool;
  const std::size_t per = (n + T - 1) / T;
  for (std::size_t t = 1; t < T; ++t)
    pool.emplace_back([&, t] { fn(std::min(n, t * per), std::min(n, (t + 1) * per)); });
  fn(0, std::min(n, per));
  for (auto& th : pool) th.join();
}

// Device copies of rule sets (for verify_hits / run_engine_scan) keyed by
// their content: a pattern's bytes are uploaded by POSITION, as verify_hits
// looks them up (rules.patterns.at(hit.pattern_id), verify.hpp:78), and the
// automaton run_engine_scan builds from the same rules is cached with them,
// so repeated scans with one RuleSet upload nothing.  A small LRU, process-wide.
struct RulesEntry {
  std::string key;
  glop_rules* rules = nullptr;
  glop_trie* trie = nullptr;  // failureless trie over truncate_prefixes(rules, prefix_len), when built
  ~RulesEntry() {
    if (trie) glop_trie_destroy(trie);
    if (rules) glop_rules_destroy(rules);
  }
};

inline std::string rules_key(const RuleSet& rules, std::size_t prefix_len) {
  std::string key = std::to_string(prefix_len) + ":" + std::to_string(rules.patterns.size()) + ":";
  for (const Pattern& p : rules.patterns) {
    key += std::to_string(p.bytes.size()) + ",";
    key += p.bytes;
  }
  return key;
}

inline std::shared_ptr<RulesEntry> device_rules(const RuleSet& rules, std::size_t prefix_len) {
  static std::mutex mu;
  static std::vector<std::shared_ptr<RulesEntry>> lru;  // most recent last
  std::string key = rules_key(rules, prefix_len);
  std::lock_guard<std::mutex> lk(mu);
  for (std::size_t i = 0; i < lru.size(); ++i)
    if (lru[i]->key == key) {
      auto e = lru[i];
      lru.erase(lru.begin() + static_cast<std::ptrdiff_t>(i));
      lru.push_back(e);
      return e;
    }
  std::string blob;
  std::vector<std::uint64_t> off{0};
  for (const Pattern& p : rules.patterns) {
    blob += p.bytes;
    off.push_back(blob.size());
  }
  auto e = std::make_shared<RulesEntry>();
  e->key = std::move(key);
  check(glop_rules_upload(context(), reinterpret_cast<const std::uint8_t*>(blob.data()), off.data(),
                          static_cast<std::uint32_t>(rules.patterns.size()), prefix_len, &e->rules),
        "verify_hits");
  lru.push_back(e);
  if (lru.size() > 16) lru.erase(lru.begin());
  return e;
}

}  // namespace logtrawl::detail

namespace logtrawl {
inline detail::DeviceTrieCache::~DeviceTrieCache() {
  if (trie) glop_trie_destroy(trie);
}
}  // namespace logtrawl
