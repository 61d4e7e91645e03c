// logtrawl -- the reference's command-line tool (tools/logtrawl.cpp:153-208)
// over the B200 path: `scan` (JSONL / summary alerts, exit 0 = no match,
// 1 = match, 2 = error), `bench` (throughput CSV, bench.hpp:140-157) and
// `gen` (reference corpus + SHA-256, loggen.hpp:44-57).  `scan` with a pfac
// engine reads each log in 64 MiB windows through the device stream
// (StreamScan) instead of loading the whole file.  Same options and
// output contract (tests/cli_test.sh of the reference, restated in
// tests/test_cli.py); CLI11 is not available here, so the option parsing is
// a small hand-written subset of what the reference's CLI11 setup accepts.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "logtrawl/jsonl.hpp"
#include "logtrawl/pipeline.hpp"
#include "workload.hpp"

namespace {

// Whole file into memory (rule files; the kmp and ac_chunked engines).
std::string slurp(const std::string& path) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw std::runtime_error("cannot open " + path);
  std::string data;
  char buf[1 << 16];
  for (size_t got; (got = std::fread(buf, 1, sizeof buf, f)) > 0;) data.append(buf, got);
  const bool bad = std::ferror(f);
  std::fclose(f);
  if (bad) throw std::runtime_error("read error on " + path);
  return data;
}

void spill(const std::string& path, const std::string& data) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw std::runtime_error("cannot open " + path + " for writing");
  const size_t put = std::fwrite(data.data(), 1, data.size(), f);
  const bool bad = std::fclose(f) != 0 || put != data.size();
  if (bad) throw std::runtime_error("short write to " + path);
}

// LOGTRAWL_WORKERS (a positive count) or 0 = the library's own parallelism
// (the reference's default_workers contract, logtrawl.cpp:36-42).
unsigned env_workers() {
  const char* env = std::getenv("LOGTRAWL_WORKERS");
  const long v = env ? std::strtol(env, nullptr, 10) : 0;
  return v > 0 ? static_cast<unsigned>(v) : 0u;
}

// A log file scanned window by window through the device stream (pfac
// engines): the file is never held whole in memory.
logtrawl::ScanReport scan_file_streamed(const std::string& path, const logtrawl::RuleSet& rules,
                                        const logtrawl::EngineConfig& cfg) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw std::runtime_error("cannot open " + path);
  logtrawl::StreamScan stream(rules, cfg, true);
  const char* env = std::getenv("LOGTRAWL_READ_WINDOW");  // tests: small reads
  std::vector<char> window(env && std::atol(env) > 0 ? std::atol(env) : (64l << 20));
  for (size_t got; (got = std::fread(window.data(), 1, window.size(), f)) > 0;)
    stream.feed(std::string_view(window.data(), got));
  const bool bad = std::ferror(f);
  std::fclose(f);
  if (bad) throw std::runtime_error("read error on " + path);
  return stream.finish();
}

// --- SHA-256 (FIPS 180-4), for the `gen` digest line -----------------------
struct Sha256 {
  uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
  static uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }
  void block(const uint8_t* p) {
    static const uint32_t k[64] = {
        0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
        0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
        0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
        0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
        0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
        0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
        0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
        0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};
    uint32_t w[64];
    for (int i = 0; i < 16; ++i) w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 | (uint32_t)p[4 * i + 2] << 8 | p[4 * i + 3];
    for (int i = 16; i < 64; ++i) {
      const uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
      const uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
      w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    for (int i = 0; i < 64; ++i) {
      const uint32_t t1 = hh + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + k[i] + w[i];
      const uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
      hh = g, g = f, f = e, e = d + t1, d = c, c = b, b = a, a = t1 + t2;
    }
    h[0] += a, h[1] += b, h[2] += c, h[3] += d, h[4] += e, h[5] += f, h[6] += g, h[7] += hh;
  }
  std::string hex(const std::string& data) {
    const uint64_t n = data.size();
    const uint8_t* p = reinterpret_cast<const uint8_t*>(data.data());
    uint64_t i = 0;
    for (; i + 64 <= n; i += 64) block(p + i);
    uint8_t tail[128] = {};
    const uint64_t r = n - i;
    memcpy(tail, p + i, r);
    tail[r] = 0x80;
    const uint64_t tl = r + 9 <= 64 ? 64 : 128, bits = n * 8;
    for (int k = 0; k < 8; ++k) tail[tl - 1 - k] = (uint8_t)(bits >> (8 * k));
    block(tail);
    if (tl == 128) block(tail + 64);
    char buf[65];
    for (int k = 0; k < 8; ++k) std::snprintf(buf + 8 * k, 9, "%08x", h[k]);
    return std::string(buf, 64);
  }
};

// --- option parsing -----------------------------------------------------------
struct Opts {
  std::vector<std::string> positional;
  std::vector<std::pair<std::string, std::string>> named;  // (--name, value)
  std::vector<std::string> flags;
};

Opts parse(int argc, char** argv, int from, const std::vector<std::string>& flag_names,
           const std::vector<std::string>& value_names) {
  Opts o;
  for (int i = from; i < argc; ++i) {
    std::string a = argv[i], v;
    const auto eq = a.find('=');
    if (a.size() > 1 && a[0] == '-' && eq != std::string::npos) v = a.substr(eq + 1), a = a.substr(0, eq);
    bool is_flag = false, is_value = false;
    for (const auto& f : flag_names) is_flag |= a == f;
    for (const auto& f : value_names) is_value |= a == f;
    if (is_flag) {
      o.flags.push_back(a);
    } else if (is_value) {
      if (eq == std::string::npos) {
        if (i + 1 >= argc) throw std::invalid_argument(a + " needs a value");
        v = argv[++i];
      }
      o.named.emplace_back(a, v);
    } else if (a.size() > 1 && a[0] == '-') {
      throw std::invalid_argument("unknown option " + a);
    } else {
      o.positional.push_back(a);
    }
  }
  return o;
}

const std::string* get(const Opts& o, std::initializer_list<const char*> names) {
  const std::string* r = nullptr;
  for (const auto& [k, v] : o.named)
    for (const char* n : names)
      if (k == n) r = &v;
  return r;
}

uint64_t to_u64(const std::string& s) {
  size_t pos = 0;
  const unsigned long long v = std::stoull(s, &pos);
  if (pos != s.size()) throw std::invalid_argument("not a number: " + s);
  return v;
}

// --- subcommands ------------------------------------------------------------------
int do_scan(const Opts& o) {  // logtrawl.cpp:54-84
  using namespace logtrawl;
  const std::string* rules_path = get(o, {"-r", "--rules"});
  if (!rules_path || o.positional.empty()) throw std::invalid_argument("scan: -r RULES and input files required");
  RuleSet rules = parse_rules(slurp(*rules_path));
  if (rules.patterns.empty()) throw std::runtime_error(*rules_path + ": rule file has no rules");
  const std::string engine_s = get(o, {"--engine"}) ? *get(o, {"--engine"}) : "pfac_compact";
  const auto engine = engine_from_name(engine_s);
  if (!engine) throw std::runtime_error("unknown engine " + engine_s);
  EngineConfig cfg;
  cfg.engine = *engine;
  if (auto* v = get(o, {"--prefix-len"})) cfg.prefix_len = to_u64(*v);
  cfg.workers = get(o, {"--workers"}) ? (unsigned)to_u64(*get(o, {"--workers"})) : env_workers();
  if (auto* v = get(o, {"--chunk-size"})) cfg.chunk_size = to_u64(*v);
  const std::string format = get(o, {"--format"}) ? *get(o, {"--format"}) : "jsonl";
  if (format != "jsonl" && format != "summary") throw std::invalid_argument("--format: jsonl|summary");
  std::size_t total = 0;
  const bool pfac = cfg.engine == EngineKind::pfac_dense || cfg.engine == EngineKind::pfac_compact;
  for (const std::string& path : o.positional) {
    ScanReport report;
    if (pfac) {
      report = scan_file_streamed(path, rules, cfg);
    } else {
      const std::string text = slurp(path);
      LineIndex lines(text);
      report = run_engine_scan(text, rules, cfg, &lines);
    }
    total += report.total_matches;
    if (format == "jsonl") {
      std::cout << render_alerts_jsonl(path, report);
    } else {
      std::cout << path << ": total_matches=" << report.total_matches << " stage1_hits=" << report.stage1_hits
                << " stage1_rejected=" << report.stage1_rejected << " bytes_scanned=" << report.bytes_scanned
                << "\n";
    }
  }
  return total ? 1 : 0;
}

int do_bench(const Opts& o) {  // logtrawl.cpp:99-129, bench.hpp:64-157
  using namespace logtrawl;
  const std::string* in = get(o, {"-i", "--input"});
  if (!in) throw std::invalid_argument("bench: -i INPUT required");
  const std::string text = slurp(*in);
  const std::string engine_s = get(o, {"--engine"}) ? *get(o, {"--engine"}) : "pfac_compact";
  const auto engine = engine_from_name(engine_s);
  if (!engine) throw std::runtime_error("unknown engine " + engine_s);
  std::vector<std::size_t> counts{10, 100, 1000};
  if (auto* v = get(o, {"--patterns"})) {
    counts.clear();
    std::stringstream ss(*v);
    for (std::string x; std::getline(ss, x, ',');) counts.push_back(to_u64(x));
  }
  const std::size_t runs = get(o, {"--runs"}) ? to_u64(*get(o, {"--runs"})) : 100;
  if (runs < 1) throw std::invalid_argument("measure: runs must be >= 1");
  const std::size_t prefix_len = get(o, {"--prefix-len"}) ? to_u64(*get(o, {"--prefix-len"})) : kDefaultPrefixLen;
  const std::size_t pattern_len = get(o, {"--pattern-len"}) ? to_u64(*get(o, {"--pattern-len"})) : 16;
  const uint32_t seed = get(o, {"--seed"}) ? (uint32_t)to_u64(*get(o, {"--seed"})) : 1;
  std::vector<EngineKind> engines{*engine};
  for (const auto& f : o.flags)
    if (f == "--paired-backends")
      engines.push_back(*engine == EngineKind::pfac_dense ? EngineKind::pfac_compact : EngineKind::pfac_dense);
  std::string csv = "engine,backend,patterns,bytes,runs,mean_seconds,throughput_bps\n";
  for (EngineKind e : engines) {
    uint32_t point = 0;
    for (std::size_t k : counts) {
      RuleSet rules;
      for (const std::string& b : glop_workload::reference_random_rules(k, pattern_len, seed + point++)) {
        Pattern p;
        p.id = (uint32_t)rules.patterns.size();
        p.name = "rand-" + std::to_string(p.id);
        p.bytes = b;
        rules.max_len = std::max(rules.max_len, b.size());
        rules.patterns.push_back(std::move(p));
      }
      // prebuilt outside the clock, one untimed warm-up (bench.hpp:35-58)
      const PrefixSet prefixes = truncate_prefixes(rules, prefix_len);
      const Automaton trie = build_failureless_trie(prefixes, e == EngineKind::pfac_dense ? Backend::dense : Backend::compact);
      EngineConfig cfg;
      cfg.engine = e;
      cfg.prefix_len = prefix_len;
      auto once = [&] {
        if (e == EngineKind::kmp) return kmp_multi(text, rules).size();
        if (e == EngineKind::ac_chunked) return run_engine_scan(text, rules, cfg).alerts.size();
        return verify_hits(text, pfac_scan(text, trie), prefixes, rules).size();
      };
      once();
      double total = 0;
      for (std::size_t r = 0; r < runs; ++r) {
        const auto t0 = std::chrono::steady_clock::now();
        volatile std::size_t sink = once();
        (void)sink;
        total += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      }
      const double mean = total / runs;
      char buf[256];
      const char* eng = (e == EngineKind::pfac_dense || e == EngineKind::pfac_compact) ? "pfac" : engine_name(e);
      const char* backend = e == EngineKind::pfac_dense ? "dense" : e == EngineKind::pfac_compact ? "compact"
                                                                 : e == EngineKind::kmp ? "-" : "dense";
      std::snprintf(buf, sizeof buf, "%s,%s,%zu,%zu,%zu,%.9g,%.9g\n", eng, backend, k, text.size(), runs, mean,
                    8.0 * text.size() / mean);
      csv += buf;
    }
  }
  if (auto* out = get(o, {"-o", "--out"})) spill(*out, csv);
  else std::cout << csv;
  return 0;
}

int do_gen(const Opts& o) {  // logtrawl.cpp:138-149
  const std::string* size = get(o, {"--size"});
  const std::string* seed = get(o, {"--seed"});
  const std::string* out = get(o, {"-o", "--out"});
  if (!size || !seed || !out) throw std::invalid_argument("gen: --size, --seed and -o required");
  const uint64_t line_len = get(o, {"--line-len"}) ? to_u64(*get(o, {"--line-len"})) : 80;
  const uint64_t n = to_u64(*size);
  if (n == 0) throw std::invalid_argument("generate_log: size is 0");
  if (line_len < 2) throw std::invalid_argument("generate_log: line_len must be >= 2");
  const std::string bytes = glop_workload::reference_generate_log(n, (uint32_t)to_u64(*seed), line_len);
  spill(*out, bytes);
  std::cout << "sha256  " << Sha256().hex(bytes) << " " << *out << " " << bytes.size() << "\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) throw std::invalid_argument("usage: logtrawl scan|bench|gen ...");
    const std::string cmd = argv[1];
    if (cmd == "scan")
      return do_scan(parse(argc, argv, 2, {}, {"-r", "--rules", "--engine", "--prefix-len", "--workers",
                                               "--chunk-size", "--format"}));
    if (cmd == "bench")
      return do_bench(parse(argc, argv, 2, {"--paired-backends"},
                            {"-i", "--input", "--engine", "--patterns", "--runs", "--prefix-len", "--pattern-len",
                             "--workers", "--seed", "-o", "--out"}));
    if (cmd == "gen") return do_gen(parse(argc, argv, 2, {}, {"--size", "--seed", "--line-len", "-o", "--out"}));
    throw std::invalid_argument("unknown subcommand " + cmd);
  } catch (const std::exception& e) {
    std::cerr << "logtrawl: " << e.what() << "\n";
    return 2;
  }
}
