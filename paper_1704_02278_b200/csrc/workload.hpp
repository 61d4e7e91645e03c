// workload.hpp -- host-side synthetic inputs: syslog corpus ranges, the
// reference's own corpus/rule generators, and the bench rule sets.
//
// Test and bench infrastructure (not the matching path).  Header-only C++17.
#pragma once
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <random>
#include <string>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "corpus.h"
#include "payload.h"

namespace glop_workload {

// Bytes [begin, begin+n) of the synthetic syslog corpus `seed`, generated on
// `threads` host threads (0 = hardware concurrency).
inline void gen_syslog(uint8_t* out, uint64_t begin, uint64_t n, uint64_t seed,
                       unsigned threads = 0) {
  using glop_corpus::kBlock;
  if (n == 0) return;
  const uint64_t b0 = begin / kBlock, b1 = (begin + n - 1) / kBlock + 1;
  if (!threads) threads = std::max(1u, std::thread::hardware_concurrency());
  threads = (unsigned)std::min<uint64_t>(threads, b1 - b0);
  auto work = [&](uint64_t lo, uint64_t hi) {
    std::vector<uint8_t> tmp(kBlock);
    for (uint64_t b = lo; b < hi; ++b) {
      glop_corpus::gen_block(tmp.data(), seed, b);
      uint64_t s = std::max(begin, b * kBlock), e = std::min(begin + n, (b + 1) * kBlock);
      memcpy(out + (s - begin), tmp.data() + (s - b * kBlock), e - s);
    }
  };
  std::vector<std::thread> pool;
  uint64_t per = (b1 - b0) / threads, extra = (b1 - b0) % threads, lo = b0;
  for (unsigned t = 0; t < threads; ++t) {
    uint64_t hi = lo + per + (t < extra ? 1 : 0);
    pool.emplace_back(work, lo, hi);
    lo = hi;
  }
  for (auto& t : pool) t.join();
}

// Bytes [begin, begin+n) of the synthetic packet-payload stream `seed`
// (payload.h), generated on `threads` host threads.
inline void gen_payload(uint8_t* out, uint64_t begin, uint64_t n, uint64_t seed, unsigned threads = 0) {
  using glop_payload::kBlock;
  if (n == 0) return;
  const uint64_t b0 = begin / kBlock, b1 = (begin + n - 1) / kBlock + 1;
  if (!threads) threads = std::max(1u, std::thread::hardware_concurrency());
  threads = (unsigned)std::min<uint64_t>(threads, b1 - b0);
  auto work = [&](uint64_t lo, uint64_t hi) {
    for (uint64_t b = lo; b < hi; ++b) {
      const uint64_t s = std::max(begin, b * kBlock), e = std::min(begin + n, (b + 1) * kBlock);
      glop_payload::gen_block_range(out + (s - begin), seed, b, (uint32_t)(s - b * kBlock),
                                    (uint32_t)(e - b * kBlock));
    }
  };
  std::vector<std::thread> pool;
  uint64_t per = (b1 - b0) / threads, extra = (b1 - b0) % threads, lo = b0;
  for (unsigned t = 0; t < threads; ++t) {
    uint64_t hi = lo + per + (t < extra ? 1 : 0);
    pool.emplace_back(work, lo, hi);
    lo = hi;
  }
  for (auto& t : pool) t.join();
}

// Snort-style content rule set for the DPI configuration: k distinct
// contents of min_len..max_len bytes: half uniformly random over the full
// byte alphabet, 45% windows of the payload stream (seed 1, first 4 MiB) whose
// 8-byte prefix occurs at most twice there (Snort contents are distinctive),
// 5% non-periodic windows of the attack strings the payloads carry (frequent
// alerts); a rejected window becomes a random content, so generation always
// terminates.
// At most 3 contents share an 8-byte prefix (stage-2 verification separates
// them).
inline std::vector<std::string> dpi_rules(size_t k, uint32_t seed, size_t min_len, size_t max_len) {
  std::vector<uint8_t> sample(4u << 20);
  gen_payload(sample.data(), 0, sample.size(), 1);
  std::vector<uint64_t> grams(sample.size() - 7);
  for (size_t i = 0; i + 8 <= sample.size(); ++i) memcpy(&grams[i], sample.data() + i, 8);
  std::sort(grams.begin(), grams.end());
  auto freq = [&](const std::string& b) {
    uint64_t g;
    memcpy(&g, b.data(), 8);
    return std::upper_bound(grams.begin(), grams.end(), g) - std::lower_bound(grams.begin(), grams.end(), g);
  };
  std::vector<std::string> attacks;
  for (const char* a = glop_payload::kAttackHost; *a;) {
    const char* e = a;
    while (*e && *e != '|') ++e;
    if ((size_t)(e - a) >= min_len) attacks.emplace_back(a, e);
    a = *e ? e + 1 : e;
  }
  std::mt19937_64 rng(seed * 0x9E3779B97F4A7C15ull + 77);
  std::unordered_set<std::string> used;
  std::unordered_map<std::string, int> per_prefix;
  std::vector<std::string> out;
  while (out.size() < k) {
    size_t len = min_len + rng() % (max_len - min_len + 1);
    std::string b;
    const size_t kind = out.size() % 20;
    if (kind < 10) {
      b.resize(len);
      for (size_t i = 0; i < len; ++i) b[i] = (char)(rng() & 0xFF);
    } else if (kind < 19) {
      b.assign(reinterpret_cast<const char*>(sample.data()) + rng() % (sample.size() - len), len);
      if (freq(b) > 2) b.clear();  // frequent protocol text: random content instead
    } else {
      const std::string& a = attacks[rng() % attacks.size()];
      len = std::min(len, a.size());
      b = a.substr(rng() % (a.size() - len + 1), len);
      bool seen[256] = {};
      int distinct = 0;
      for (size_t i = 0; i < 8; ++i) distinct += !seen[(uint8_t)b[i]], seen[(uint8_t)b[i]] = true;
      if (distinct < 6) b.clear();  // periodic ("../../..") windows: random content instead
    }
    if (b.empty()) {
      b.resize(len);
      for (size_t i = 0; i < len; ++i) b[i] = (char)(rng() & 0xFF);
    }
    if (used.count(b) || per_prefix[b.substr(0, 8)] >= 3) continue;
    ++per_prefix[b.substr(0, 8)];
    used.insert(b);
    out.push_back(std::move(b));
  }
  return out;
}

// Reference corpus semantics (loggen.hpp:35-57): MT19937 low-byte rejection
// sampling onto printable ASCII, LF at every multiple of line_len.
inline char printable_from(std::mt19937& rng) {
  for (;;) {
    uint32_t b = rng() & 0xFF;
    if (b < 190) return (char)(32 + b % 95);
  }
}

inline std::string reference_generate_log(uint64_t size, uint32_t seed, uint64_t line_len) {
  std::mt19937 rng(seed);
  std::string s(size, '\0');
  for (uint64_t p = 0; p < size; ++p) s[p] = (p % line_len == 0) ? '\n' : printable_from(rng);
  return s;
}

// Reference rule semantics (loggen.hpp:60-78): distinct random printable
// patterns of a fixed length.
inline std::vector<std::string> reference_random_rules(size_t count, size_t len, uint32_t seed) {
  std::mt19937 rng(seed);
  std::vector<std::string> out;
  std::unordered_set<std::string> seen;
  while (out.size() < count) {
    std::string b(len, '\0');
    for (char& c : b) c = printable_from(rng);
    if (!seen.insert(b).second) continue;
    out.push_back(std::move(b));
  }
  return out;
}

// All distinct 8-byte windows of the literal text of the incident templates
// (weight class <= 'c'), taken after the '^' marker, never spanning a
// placeholder, and never occurring in the literal text of a routine
// (non-incident) template -- so vocabulary rules fire on incident lines only.
// Deterministic order (template order, then position).
inline std::vector<std::string> vocab_windows(size_t w = 8) {
  std::vector<std::string> out;
  std::unordered_set<std::string> seen;
  std::string routine;  // literal text of every routine template
  for (const char* p = glop_corpus::kTplHost; *p;) {
    const char* e = p;
    while (*e && *e != '|') ++e;
    if (*p > 'c') {
      for (const char* x = p + 1; x < e; ++x) {
        if (*x == '{') {
          routine += '\x01';
          while (x < e && *x != '}') ++x;
        } else if (*x != '^') {
          routine += *x;
        }
      }
      routine += '\x01';
    }
    p = *e ? e + 1 : e;
  }
  const char* p = glop_corpus::kTplHost;
  while (*p) {
    const char* e = p;
    while (*e && *e != '|') ++e;
    std::string tpl(p + 1, e);
    bool incident = *p <= 'c';
    p = *e ? e + 1 : e;
    size_t caret = tpl.find('^');
    if (!incident || caret == std::string::npos) continue;
    std::string body = tpl.substr(caret + 1);
    std::string seg;
    auto flush = [&]() {
      for (size_t i = 0; i + w <= seg.size(); ++i) {
        std::string win = seg.substr(i, w);
        if (routine.find(win) != std::string::npos) continue;
        if (seen.insert(win).second) out.push_back(win);
      }
      seg.clear();
    };
    for (size_t i = 0; i < body.size(); ++i) {
      if (body[i] == '{') {
        flush();
        i = body.find('}', i);
      } else if (body[i] != '^') {
        seg.push_back(body[i]);
      }
    }
    flush();
  }
  return out;
}

struct Rule {
  std::string name;
  std::string bytes;
};

// Bench / parity rule set: k - k/2 random printable patterns with the
// reference's random_rules semantics, plus k/2 windows sampled from the
// incident vocabulary (falls back to more random patterns if the pool is
// exhausted).  All patterns are distinct.
inline std::vector<Rule> synthetic_rules(size_t k, uint32_t seed, size_t len = 8) {
  size_t k_vocab = k / 2;
  std::vector<std::string> pool = vocab_windows(len);
  std::mt19937 rng(seed ^ 0x9e3779b9u);
  for (size_t i = pool.size(); i > 1; --i) std::swap(pool[i - 1], pool[rng() % i]);
  if (k_vocab > pool.size()) k_vocab = pool.size();
  std::vector<std::string> rnd = reference_random_rules(k + k_vocab, len, seed);
  std::unordered_set<std::string> used;
  std::vector<Rule> rules;
  size_t ri = 0, vi = 0;
  // interleave so prefix subsets of the list stay mixed
  while (rules.size() < k) {
    bool take_vocab = vi < k_vocab && (rules.size() % 2 == 1 || ri >= rnd.size());
    std::string b = take_vocab ? pool[vi++] : rnd[ri++];
    if (!used.insert(b).second) continue;
    Rule r;
    r.name = (take_vocab ? "vocab-" : "rand-") + std::to_string(rules.size());
    r.bytes = std::move(b);
    rules.push_back(std::move(r));
    if (ri >= rnd.size() && vi >= k_vocab && rules.size() < k) {
      rnd = reference_random_rules(rnd.size() * 2, len, seed + 1);
      ri = 0;
    }
  }
  return rules;
}

}  // namespace glop_workload
