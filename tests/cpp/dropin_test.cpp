// Drop-in API test: the reference's C++ call sites compiled unchanged against
// include/logtrawl/ (this repo) and run on the B200 through libglop.so.
// Each check restates a reference test (file:line under
// /root/reference/proj/tests/).  Exit status = number of failed checks.
#include <cstdio>
#include <random>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "logtrawl/pipeline.hpp"

using namespace logtrawl;

static int failures = 0;
#define CHECK(cond)                                                  \
  do {                                                               \
    if (!(cond)) {                                                   \
      ++failures;                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);    \
    }                                                                \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static RuleSet make_rules(const std::vector<std::string>& pats) {
  RuleSet r;
  for (const std::string& b : pats) {
    r.patterns.push_back({static_cast<std::uint32_t>(r.patterns.size()), "p" + std::to_string(r.patterns.size()), b});
    r.max_len = std::max(r.max_len, b.size());
  }
  return r;
}

static std::vector<Match> matches_of(const std::vector<Alert>& alerts) {
  std::vector<Match> out;
  for (const Alert& a : alerts) out.push_back({a.offset, a.rule_id});
  return out;
}

// brute force, independent of the code under test
static std::vector<Match> brute(const std::string& text, const RuleSet& r) {
  std::vector<Match> out;
  for (const Pattern& p : r.patterns)
    for (std::size_t i = 0; i + p.bytes.size() <= text.size(); ++i)
      if (text.compare(i, p.bytes.size(), p.bytes) == 0) out.push_back({i, p.id});
  std::sort(out.begin(), out.end());
  return out;
}

int main() {
  // test_scan.cpp:57-78
  {
    RuleSet r = make_rules({"HIS", "SHE"});
    auto hits = pfac_scan("SHIS", build_failureless_trie(truncate_prefixes(r, 8)), {.workers = 1});
    CHECK(hits.size() == 1 && hits[0] == (Hit{1, 0, 3}));
    RuleSet ab = make_rules({"AB", "ABC"});
    CHECK(pfac_scan("ABAB", build_failureless_trie(truncate_prefixes(ab, 8))) ==
          (std::vector<Hit>{{0, 0, 2}, {2, 0, 2}}));
    CHECK(pfac_scan("", build_failureless_trie(truncate_prefixes(make_rules({"A"}), 8))).empty());
    CHECK(throws<std::invalid_argument>([&] { pfac_scan("x", build_ac_automaton(make_rules({"A"}))); }));
  }
  // test_automaton.cpp:55-102
  {
    Automaton a = build_failureless_trie(truncate_prefixes(make_rules({"HIS", "SHE"}), 8));
    CHECK(a.state_count == 7);
    CHECK(build_failureless_trie(truncate_prefixes(make_rules({"AB", "ABC"}), 8)).state_count == 4);
    CHECK(build_failureless_trie(PrefixSet{}).state_count == 1);
    CHECK(throws<CapacityError>(
        [&] { build_failureless_trie(truncate_prefixes(make_rules({"ABCDEFGH"}), 8), Backend::dense, 4); }));
    Automaton c = to_compact(a);
    CHECK(c.table_bytes() == 7 * sizeof(Automaton::CompactNode) + 6 * sizeof(std::int32_t));
    CHECK(a.dump().find("0 --72--> 1") != std::string::npos);
  }
  // test_verify.cpp:26-65
  {
    RuleSet r = make_rules({"GETPASSWORDFILE"});
    PrefixSet ps = truncate_prefixes(r, 8);
    auto ok = verify_hits("0123456789GETPASSWORDFILE....", {{10, 0, 8}}, ps, r);
    CHECK(ok.size() == 1 && ok[0].offset == 10 && ok[0].pattern_len == 15 && ok[0].verified);
    CHECK(verify_hits("0123456789GETPASSWXYZ..........", {{10, 0, 8}}, ps, r).empty());
    RuleSet root = make_rules({"root"});
    CHECK(verify_hits("rootkit", {{0, 0, 4}}, truncate_prefixes(root, 8), root).size() == 1);
    CHECK(verify_hits("..GETPASSW", {{2, 0, 8}}, ps, r).empty());
    CHECK(throws<std::logic_error>([&] { verify_hits("ab", {{1, 0, 4}}, truncate_prefixes(root, 8), root); }));
    ScanReport rep = assemble_report(std::vector<Alert>(3), 5, 1000);
    CHECK(rep.total_matches == 3 && rep.stage1_rejected == 2 && rep.bytes_scanned == 1000);
  }
  // test_verify.cpp:114-124
  {
    LineIndex idx("abc\ndef\n\nxyz");
    CHECK(idx.line_count() == 4 && idx.line_of(0) == 1 && idx.line_of(3) == 1 && idx.line_of(4) == 2 &&
          idx.line_of(8) == 3 && idx.line_of(9) == 4 && idx.line_begin(2) == 4);
  }
  // test_kmp.cpp:29-74
  {
    CHECK(build_failure_table({0, "p", "ABAB"}).table == (std::vector<std::uint32_t>{0, 0, 1, 2}));
    Pattern aab{0, "p", "AAB"}, his{0, "p", "HIS"}, aa{0, "p", "AA"};
    CHECK(kmp_search("AABAABAAB", aab, build_failure_table(aab)) == (std::vector<std::size_t>{0, 3, 6}));
    CHECK(kmp_search("SHIS", his, build_failure_table(his)) == (std::vector<std::size_t>{1}));
    CHECK(kmp_search("AB", his, build_failure_table(his)).empty());
    CHECK(kmp_search("AAAA", aa, build_failure_table(aa)) == (std::vector<std::size_t>{0, 1, 2}));
    RuleSet r = make_rules({"HIS", "SHE"});
    CHECK(kmp_multi("SHIS", r) == (std::vector<Match>{{1, 0}}));
  }
  // test_rules.cpp:275-323
  {
    RuleSet r = parse_rules("ssh-fail : HIS\nshell : SHE");
    CHECK(r.patterns.size() == 2 && r.patterns[1].name == "shell" && r.max_len == 3);
    CHECK(parse_rules("# comment\n\nr : \\x41\\x42").patterns[0].bytes == "AB");
    CHECK(throws<RuleParseError>([] { parse_rules("a : X\nb : X"); }));
    CHECK(throws<RuleParseError>([] { parse_rules("a : \\xZZ"); }));
    try {
      parse_rules("a : X\n# c\nb : X");
      CHECK(false);
    } catch (const RuleParseError& e) {
      CHECK(e.line() == 3 && std::string(e.what()).find("line 1") != std::string::npos);
    }
    CHECK(truncate_prefixes(parse_rules("x : ABCDEFGHX\ny : ABCDEFGHY"), 8).entries.size() == 1);
    CHECK(throws<std::invalid_argument>([] { truncate_prefixes(RuleSet{}, 0); }));
  }
  // test_scan.cpp:157-176 + acceptance.cpp:42-78 (reduced): every engine
  // equals brute force on random inputs; workers never matter
  {
    std::mt19937 rng(2024);
    for (int trial = 0; trial < 60; ++trial) {
      const bool full = trial % 2;
      std::set<std::string> used;
      std::vector<std::string> pats;
      const std::size_t count = 1 + rng() % 32;
      while (pats.size() < count) {
        std::string b;
        const std::size_t len = 1 + rng() % 16;
        for (std::size_t j = 0; j < len; ++j) b.push_back(full ? char(rng() & 0xFF) : char('A' + rng() % 4));
        if (used.insert(b).second) pats.push_back(b);
      }
      std::string text;
      const std::size_t n = rng() % 4096;
      for (std::size_t i = 0; i < n; ++i) text.push_back(full ? char(rng() & 0xFF) : char('A' + rng() % 4));
      RuleSet r = make_rules(pats);
      const auto truth = brute(text, r);
      for (std::size_t L : {4u, 8u, 4096u}) {
        PrefixSet ps = truncate_prefixes(r, L);
        for (Backend b : {Backend::dense, Backend::compact}) {
          auto hits = pfac_scan(text, build_failureless_trie(ps, b), {.workers = static_cast<unsigned>(1 + rng() % 4)});
          CHECK(matches_of(verify_hits(text, hits, ps, r)) == truth);
        }
      }
      for (EngineKind e : {EngineKind::kmp, EngineKind::pfac_dense, EngineKind::pfac_compact, EngineKind::ac_chunked}) {
        EngineConfig cfg;
        cfg.engine = e;
        CHECK(matches_of(run_engine_scan(text, r, cfg).alerts) == truth);
      }
      CHECK(naive_scan(text, r) == truth);
    }
  }
  // test_scan.cpp:90-146 / acceptance.cpp:80-93: chunked AC, the boundary
  // problem and its overlap fix, on the device
  {
    RuleSet r = make_rules({"HIS", "SHE"});
    Automaton ac = build_ac_automaton(r);
    const std::string text = "XXHISXX";
    auto lost = chunked_ac_scan(text, ac, {.workers = 1, .chunk_size = 4, .overlap = 0});
    CHECK(lost.empty());
    auto found = chunked_ac_scan(text, ac, {.workers = 1, .chunk_size = 4, .overlap = 2});
    CHECK(found == (std::vector<Match>{{2, 0}}));
    CHECK(found == chunked_ac_scan(text, ac, {.workers = 1, .chunk_size = text.size(), .overlap = 0}));
    Automaton aba = build_ac_automaton(make_rules({"ABA"}));
    auto whole = chunked_ac_scan("ABABA", aba, {.workers = 1, .chunk_size = 5, .overlap = 0});
    CHECK(whole == (std::vector<Match>{{0, 0}, {2, 0}}));
    for (std::size_t ov : {0u, 1u, 10u}) CHECK(chunked_ac_scan("ABABA", aba, {.chunk_size = 100, .overlap = ov}) == whole);
    CHECK(throws<std::invalid_argument>([&] {
      chunked_ac_scan("x", build_failureless_trie(truncate_prefixes(r, 8)), {});
    }));
    // random inputs, lossless (overlap >= max_len - 1) and lossy overlaps,
    // against the ownership rule restated by brute force (scan.hpp:224-233)
    std::mt19937 rng(13);
    for (int trial = 0; trial < 100; ++trial) {
      const bool full = trial % 2;
      std::set<std::string> used;
      std::vector<std::string> pats;
      while (pats.size() < 8) {
        std::string b;
        const std::size_t len = 1 + rng() % 8;
        for (std::size_t j = 0; j < len; ++j) b.push_back(full ? char(rng() & 0xFF) : char('A' + rng() % 4));
        if (used.insert(b).second) pats.push_back(b);
      }
      std::string text;
      for (std::size_t i = 0; i < 2048; ++i) text.push_back(full ? char(rng() & 0xFF) : char('A' + rng() % 4));
      RuleSet rr = make_rules(pats);
      Automaton a = build_ac_automaton(rr, trial % 3 ? Backend::dense : Backend::compact);
      const auto truth = brute(text, rr);
      CHECK(chunked_ac_scan(text, a, {.chunk_size = text.size(), .overlap = 0}) == truth);
      const std::size_t chunk = 1 + rng() % 64;
      const std::size_t overlap = trial % 4 == 3 ? rng() % rr.max_len : rr.max_len - 1 + rng() % 8;
      std::vector<Match> expect;
      for (const Match& m : truth) {
        const std::size_t own = m.offset / chunk * chunk;
        if (m.offset + rr.patterns[m.pattern_id].bytes.size() <= std::min(own + chunk + overlap, text.size()))
          expect.push_back(m);
      }
      CHECK(chunked_ac_scan(text, a, {.workers = static_cast<unsigned>(1 + rng() % 8), .chunk_size = chunk, .overlap = overlap}) == expect);
      if (overlap >= rr.max_len - 1) CHECK(expect == truth);
    }
  }
  // run_engine_scan with a LineIndex: lines from the device pipeline equal the
  // host index (pipeline.hpp:49-100, verify.hpp:40-64); stage-1 counts
  {
    std::string text;
    std::mt19937 rng(77);
    for (int i = 0; i < 20000; ++i) text += (rng() % 5 == 0) ? "Failed password for root\n" : "ok line " + std::to_string(rng()) + "\n";
    RuleSet r = make_rules({"Failed password for root", "ok line 1", "ok line 12", "root\nok"});
    LineIndex idx(text);
    for (EngineKind e : {EngineKind::pfac_dense, EngineKind::pfac_compact}) {
      EngineConfig cfg;
      cfg.engine = e;
      ScanReport rep = run_engine_scan(text, r, cfg, &idx);
      CHECK(matches_of(rep.alerts) == brute(text, r));
      bool lines_ok = !rep.alerts.empty();
      for (const Alert& a : rep.alerts) lines_ok = lines_ok && a.line == idx.line_of(a.offset) && a.line > 0;
      CHECK(lines_ok);
      const PrefixSet ps = truncate_prefixes(r, cfg.prefix_len);
      CHECK(rep.stage1_hits == pfac_scan(text, build_failureless_trie(ps)).size());
      CHECK(rep.stage1_rejected == rep.stage1_hits - rep.total_matches && rep.bytes_scanned == text.size());
      // a LineIndex of another text keeps its own answers
      LineIndex other("a\nb\n");
      for (const Alert& a : run_engine_scan(text, r, cfg, &other).alerts) lines_ok = lines_ok && a.line == other.line_of(a.offset);
      CHECK(lines_ok);
    }
  }
  // verify_hits looks patterns up by position and reports their ids
  // (verify.hpp:78, :91): a RuleSet whose ids are not positions
  {
    RuleSet r;
    r.patterns = {{7, "seven", "GETPASSWORD"}, {3, "three", "root"}};
    r.max_len = 11;
    PrefixSet ps = truncate_prefixes(make_rules({"GETPASSWORD", "root"}), 8);
    auto al = verify_hits("rootGETPASSWORD", {{0, 1, 4}, {4, 0, 8}}, ps, r);
    CHECK(al.size() == 2 && al[0].rule_id == 3 && al[0].rule_name == "three" && al[1].rule_id == 7 &&
          al[1].pattern_len == 11);
    auto same_off = verify_hits("rootroot", {{0, 0, 4}, {0, 1, 4}}, truncate_prefixes(make_rules({"root", "root"}), 8),
                                RuleSet{{{9, "a", "root"}, {2, "b", "root"}}, 4});
    CHECK(same_off.size() == 2 && same_off[0].rule_id == 2 && same_off[1].rule_id == 9);  // sorted by (offset, rule_id)
    CHECK(throws<std::logic_error>([&] { verify_hits("rootroot", {{0, 5, 4}}, ps, r); }));  // patterns.at()
  }
  // kmp_search runs the given failure table as the reference does, canonical
  // or not (kmp.hpp:41-69), and long patterns
  {
    auto seq = [](const std::string& t, const std::string& p, const std::vector<std::uint32_t>& tab, std::uint64_t& cmp) {
      std::vector<std::size_t> out;
      std::size_t j = 0;
      for (std::size_t i = 0; i < t.size(); ++i)
        for (;;) {
          ++cmp;
          if (t[i] == p[j]) {
            if (++j == p.size()) out.push_back(i + 1 - p.size()), j = tab[p.size() - 1];
            break;
          }
          if (j == 0) break;
          j = tab[j - 1];
        }
      return out;
    };
    const std::string text = "AABAABAABAAAABAABAAB";
    Pattern aab{0, "p", "AAB"};
    FailureTable zero{0, {0, 0, 0}};
    std::uint64_t c1 = 0, c2 = 0;
    CHECK(kmp_search(text, aab, zero, &c1) == seq(text, "AAB", zero.table, c2) && c1 == c2);
    std::string lp(9000, 'x');
    lp.back() = 'y';
    std::string lt = std::string(20000, 'x') + "y" + lp + "zz";
    Pattern longp{0, "L", lp};
    FailureTable ft = build_failure_table(longp);
    c1 = c2 = 0;
    CHECK(kmp_search(lt, longp, ft, &c1) == seq(lt, lp, ft.table, c2) && c1 == c2 && c1 > 0);
  }
  // concurrent callers (the reference is reentrant): threads
  // scanning at once with one shared rule set and automaton get the results
  // a single caller gets
  {
    std::mt19937 rng(99);
    std::vector<std::string> texts(6);
    for (auto& t : texts)
      for (int i = 0; i < 40000; ++i) t += (rng() % 7 == 0) ? "Failed password for root\n" : "x" + std::to_string(rng()) + "\n";
    RuleSet r = make_rules({"Failed password", "password for", "root\nx1", "x12", "x999"});
    const Automaton shared = build_failureless_trie(truncate_prefixes(r, 8));
    std::vector<std::vector<Match>> want;
    std::vector<std::size_t> want_hits;
    for (const auto& t : texts) {
      want.push_back(brute(t, r));
      want_hits.push_back(pfac_scan(t, shared).size());
    }
    std::vector<int> ok(texts.size() * 3, 0);
    std::vector<std::thread> pool;
    for (std::size_t w = 0; w < 3; ++w)
      pool.emplace_back([&, w] {
        for (std::size_t i = 0; i < texts.size(); ++i) {
          EngineConfig cfg;
          cfg.engine = (i + w) % 2 ? EngineKind::pfac_dense : EngineKind::pfac_compact;
          const bool a = matches_of(run_engine_scan(texts[i], r, cfg).alerts) == want[i];
          const bool b = pfac_scan(texts[i], shared).size() == want_hits[i];
          ok[w * texts.size() + i] = a && b;
        }
      });
    for (auto& t : pool) t.join();
    bool all = true;
    for (int v : ok) all = all && v;
    CHECK(all);
  }
  std::printf("%s (%d failure%s)\n", failures ? "FAILED" : "OK", failures, failures == 1 ? "" : "s");
  return failures;
}
