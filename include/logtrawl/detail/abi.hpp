#pragma once
// Glue between the drop-in C++ API and the C ABI (include/glop.h): the
// process-wide device group, content-keyed device copies of rule sets, and
// the mapping of glop_status codes onto the exception types the reference
// throws.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <memory>
#include <atomic>
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

// The device group the drop-in API runs on -- every visible GPU by default,
// as the reference's scans use every hardware thread (scan.hpp:182-195,
// default_workers).  GLOP_DEVICES="0,2,3" picks devices (a device may repeat:
// N contexts on one GPU); GLOP_DEVICE=d a single one.  Each calling thread
// gets its own group (its own streams and scratch) on those devices, so
// concurrent scans run concurrently, as the reference's reentrant scans do
// (SPEC.md:163, :293); device copies of automata and rule sets are shared.
inline const std::vector<int>& group_devices() {
  static const std::vector<int> devs = [] {
    std::vector<int> d;
    if (const char* list = std::getenv("GLOP_DEVICES")) {
      for (const char* c = list; *c;) {
        char* end = nullptr;
        const long v = std::strtol(c, &end, 10);
        if (end == c) break;
        d.push_back(static_cast<int>(v));
        c = *end == ',' ? end + 1 : end;
      }
    } else if (const char* one = std::getenv("GLOP_DEVICE")) {
      d.push_back(std::atoi(one));
    }
    return d;
  }();
  return devs;
}

struct GroupHolder {
  glop_group* g = nullptr;
  glop_status st = GLOP_OK;
  std::string err;
  GroupHolder() {
    const std::vector<int>& devs = group_devices();
    st = glop_group_create(devs.empty() ? nullptr : devs.data(), static_cast<int>(devs.size()), &g);
    if (st != GLOP_OK) err = glop_last_error();
  }
  ~GroupHolder() { glop_group_destroy(g); }
};

inline glop_group* group() {
  thread_local GroupHolder h;
  if (h.st != GLOP_OK) throw std::runtime_error("glop: no usable B200 device: " + h.err);
  return h.g;
}

// The group's first context: single-device calls (verify_hits, chunked AC).
inline glop_ctx* context() { return glop_group_ctx(group(), 0); }

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
  glop_group_rules* rules = nullptr;
  glop_group_trie* trie = nullptr;  // failureless trie over truncate_prefixes(rules, prefix_len), when built
  // alerts and text bytes of the last pipeline call: the Alert storage of a
  // similar-sized call is prepared while the device works
  std::atomic<std::uint64_t> last_alerts{0}, last_bytes{0};
  ~RulesEntry() {
    if (trie) glop_group_trie_destroy(trie);
    if (rules) glop_group_rules_destroy(rules);
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
  check(glop_group_rules_upload(group(), reinterpret_cast<const std::uint8_t*>(blob.data()), off.data(),
                                static_cast<std::uint32_t>(rules.patterns.size()), prefix_len, &e->rules),
        "verify_hits");
  lru.push_back(e);
  if (lru.size() > 16) lru.erase(lru.begin());
  return e;
}

}  // namespace logtrawl::detail

namespace logtrawl {
inline detail::DeviceTrieCache::~DeviceTrieCache() {
  if (trie) glop_group_trie_destroy(trie);
}
}  // namespace logtrawl
