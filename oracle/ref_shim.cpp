// ref_shim.cpp -- C ABI over the UNMODIFIED reference implementation.
// TEST / BASELINE INFRASTRUCTURE ONLY.
//
// Compiled against /root/reference/proj/include where it lies (nothing is
// copied) into oracle/_ref/libref_logtrawl.so by oracle/Makefile.  Used to
// pin the C restatement (oracle/pfac_oracle.c) and as the CPU baseline
// ("kind": "reference") in bench.py: the timed call is the reference's own
// measure() harness (bench.hpp:64-113) over pfac_scan + verify_hits.
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "logtrawl/bench.hpp"
#include "logtrawl/kmp.hpp"
#include "logtrawl/pipeline.hpp"
#include "workload.hpp"  // synthetic inputs (paper_1704_02278_b200/csrc), not the matching path

using namespace logtrawl;

namespace {
struct ref_hit {
  uint64_t offset;
  uint32_t pattern_id, matched_len;
};
struct ref_alert {
  uint64_t offset;
  uint32_t rule_id, pattern_len;
  uint64_t line;
};

RuleSet rules_of(const uint8_t* bytes, const uint64_t* off, uint32_t k) {
  RuleSet r;
  for (uint32_t i = 0; i < k; ++i) {
    Pattern p;
    p.id = i;
    p.name = "r" + std::to_string(i);
    p.bytes.assign((const char*)bytes + off[i], off[i + 1] - off[i]);
    r.max_len = std::max(r.max_len, p.bytes.size());
    r.patterns.push_back(std::move(p));
  }
  return r;
}
}  // namespace

extern "C" {

// truncate_prefixes -> build_failureless_trie -> pfac_scan -> verify_hits
int ref_pfac_scan_verify(const uint8_t* text, uint64_t n, const uint8_t* bytes,
                         const uint64_t* off, uint32_t k, uint64_t L, int compact,
                         unsigned workers, int with_lines, ref_hit** hits_out,
                         uint64_t* n_hits, ref_alert** alerts_out, uint64_t* n_alerts) {
  try {
    RuleSet r = rules_of(bytes, off, k);
    std::string_view tv((const char*)text, n);
    PrefixSet ps = truncate_prefixes(r, L);
    Automaton trie = build_failureless_trie(ps, compact ? Backend::compact : Backend::dense);
    auto hits = pfac_scan(tv, trie, {.workers = workers});
    LineIndex idx(tv);
    auto alerts = verify_hits(tv, hits, ps, r, with_lines ? &idx : nullptr);
    *hits_out = (ref_hit*)malloc(sizeof(ref_hit) * (hits.size() + 1));
    for (size_t i = 0; i < hits.size(); ++i)
      (*hits_out)[i] = {hits[i].offset, hits[i].pattern_id, hits[i].matched_len};
    *n_hits = hits.size();
    *alerts_out = (ref_alert*)malloc(sizeof(ref_alert) * (alerts.size() + 1));
    for (size_t i = 0; i < alerts.size(); ++i)
      (*alerts_out)[i] = {alerts[i].offset, alerts[i].rule_id, alerts[i].pattern_len,
                          alerts[i].line};
    *n_alerts = alerts.size();
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const CapacityError&) {
    return 2;
  } catch (const std::logic_error&) {
    return 3;
  } catch (...) {
    return 4;
  }
}

// The reference benchmark harness (bench.hpp:64-113): prebuilds the trie,
// one untimed warm-up, then `runs` timed pfac_scan + verify_hits (or
// kmp_multi).  engine: 0 kmp, 1 pfac_dense, 2 pfac_compact.
int ref_measure(const uint8_t* text, uint64_t n, const uint8_t* bytes, const uint64_t* off,
                uint32_t k, uint64_t L, int engine, unsigned workers, uint64_t runs,
                double* mean_seconds, double* throughput_bps) {
  try {
    RuleSet r = rules_of(bytes, off, k);
    EngineConfig cfg;
    cfg.engine = engine == 0 ? EngineKind::kmp
                             : (engine == 1 ? EngineKind::pfac_dense : EngineKind::pfac_compact);
    cfg.prefix_len = L;
    cfg.workers = workers;
    ThroughputReport rep = measure(cfg, std::string_view((const char*)text, n), r, runs);
    *mean_seconds = rep.mean_seconds;
    *throughput_bps = rep.throughput_bps;
    return 0;
  } catch (...) {
    return 4;
  }
}

// measure()'s timed body (bench.hpp:103-109: pfac_scan + verify_hits with a
// prebuilt trie) with an explicit warm-up count; per-run wall seconds.
int ref_time_pfac(const uint8_t* text, uint64_t n, const uint8_t* bytes, const uint64_t* off, uint32_t k,
                  uint64_t L, int compact, unsigned workers, uint32_t warmup, uint32_t runs,
                  double* run_seconds, uint64_t* n_alerts) {
  try {
    RuleSet r = rules_of(bytes, off, k);
    std::string_view tv((const char*)text, n);
    PrefixSet ps = truncate_prefixes(r, L);
    Automaton trie = build_failureless_trie(ps, compact ? Backend::compact : Backend::dense);
    ScanConfig sc;
    sc.workers = workers ? workers : default_workers();
    size_t na = 0;
    for (uint32_t i = 0; i < warmup + runs; ++i) {
      auto t0 = std::chrono::steady_clock::now();
      std::vector<Hit> hits = pfac_scan(tv, trie, sc);
      na = verify_hits(tv, hits, ps, r).size();
      auto t1 = std::chrono::steady_clock::now();
      if (i >= warmup) run_seconds[i - warmup] = std::chrono::duration<double>(t1 - t0).count();
    }
    *n_alerts = na;
    return 0;
  } catch (...) {
    return 4;
  }
}

// kmp_multi timed the same way (bench.hpp:83-91), single-threaded by design.
int ref_time_kmp(const uint8_t* text, uint64_t n, const uint8_t* p, uint32_t m, uint32_t warmup, uint32_t runs,
                 double* run_seconds, uint64_t* n_matches) {
  RuleSet r;
  r.patterns.push_back({0, "p", std::string((const char*)p, m)});
  r.max_len = m;
  std::vector<FailureTable> tables{build_failure_table(r.patterns[0])};
  std::string_view tv((const char*)text, n);
  for (uint32_t i = 0; i < warmup + runs; ++i) {
    auto t0 = std::chrono::steady_clock::now();
    *n_matches = kmp_multi(tv, r, &tables).size();
    auto t1 = std::chrono::steady_clock::now();
    if (i >= warmup) run_seconds[i - warmup] = std::chrono::duration<double>(t1 - t0).count();
  }
  return 0;
}

int ref_kmp_search(const uint8_t* text, uint64_t n, const uint8_t* p, uint32_t m,
                   uint64_t** offs, uint64_t* n_offs, uint64_t* comparisons) {
  Pattern pt{0, "p", std::string((const char*)p, m)};
  FailureTable ft = build_failure_table(pt);
  uint64_t cmp = 0;
  auto v = kmp_search(std::string_view((const char*)text, n), pt, ft, &cmp);
  *offs = (uint64_t*)malloc(sizeof(uint64_t) * (v.size() + 1));
  for (size_t i = 0; i < v.size(); ++i) (*offs)[i] = v[i];
  *n_offs = v.size();
  *comparisons = cmp;
  return 0;
}

unsigned ref_default_workers(void) { return default_workers(); }

// chunked_ac_scan (scan.hpp:207-243) over build_ac_automaton(rules): sorted
// (offset, pattern_id) matches as 16-byte records (offset, id, 0).
int ref_chunked_ac_scan(const uint8_t* text, uint64_t n, const uint8_t* bytes, const uint64_t* off, uint32_t k,
                        uint64_t chunk_size, uint64_t overlap, unsigned workers, ref_hit** out, uint64_t* n_out) {
  try {
    RuleSet r = rules_of(bytes, off, k);
    Automaton ac = build_ac_automaton(r);
    ScanConfig sc;
    sc.workers = workers;
    sc.chunk_size = chunk_size;
    sc.overlap = overlap;
    auto ms = chunked_ac_scan(std::string_view((const char*)text, n), ac, sc);
    *out = (ref_hit*)malloc(sizeof(ref_hit) * (ms.size() + 1));
    for (size_t i = 0; i < ms.size(); ++i) (*out)[i] = {ms[i].offset, ms[i].pattern_id, 0};
    *n_out = ms.size();
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (...) {
    return 4;
  }
}

// ---- synthetic workloads for the reference arm, so it never maps the
// product library (the same header-only generators libglop exports).
int ref_gen_syslog(uint8_t* out, uint64_t begin, uint64_t n, uint64_t seed, unsigned threads) {
  glop_workload::gen_syslog(out, begin, n, seed, threads);
  return 0;
}
int ref_gen_payload(uint8_t* out, uint64_t begin, uint64_t n, uint64_t seed, unsigned threads) {
  glop_workload::gen_payload(out, begin, n, seed, threads);
  return 0;
}
int ref_gen_rules(uint32_t k, uint32_t seed, uint32_t len, uint8_t* bytes, uint8_t* is_vocab) {
  auto rules = glop_workload::synthetic_rules(k, seed, len);
  for (uint32_t i = 0; i < k; ++i) {
    memcpy(bytes + (size_t)i * len, rules[i].bytes.data(), len);
    if (is_vocab) is_vocab[i] = rules[i].name.rfind("vocab-", 0) == 0;
  }
  return 0;
}
int ref_gen_dpi_rules(uint32_t k, uint32_t seed, uint32_t min_len, uint32_t max_len, uint8_t* bytes,
                      uint64_t* off) {
  const auto rules = glop_workload::dpi_rules(k, seed, min_len, max_len);
  uint64_t o = 0;
  for (uint32_t i = 0; i < k; ++i) {
    off[i] = o;
    memcpy(bytes + o, rules[i].data(), rules[i].size());
    o += rules[i].size();
  }
  off[k] = o;
  return 0;
}

// The CPU model of this host (cpu_baseline), from /proc/cpuinfo.
int ref_cpu_model(char* out, uint64_t cap) {
  std::string model = "unknown";
  if (FILE* f = fopen("/proc/cpuinfo", "r")) {
    char line[512];
    while (fgets(line, sizeof line, f))
      if (!strncmp(line, "model name", 10)) {
        const char* c = strchr(line, ':');
        if (c) {
          model = c + 1;
          while (!model.empty() && (model.front() == ' ' || model.front() == '\t')) model.erase(0, 1);
          while (!model.empty() && (model.back() == '\n' || model.back() == ' ')) model.pop_back();
        }
        break;
      }
    fclose(f);
  }
  snprintf(out, cap, "%s", model.c_str());
  return 0;
}

void ref_free(void* p) { free(p); }
}
