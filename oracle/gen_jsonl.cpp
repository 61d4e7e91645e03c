// gen_jsonl -- TEST INFRASTRUCTURE ONLY.  Renders the reference CLI's scan
// output (tools/logtrawl.cpp:54-84: run_engine_scan with a LineIndex, then
// render_alerts_jsonl, jsonl.hpp:14-34) with the unmodified reference
// headers (+ the nlohmann json.hpp the reference vendors), for the CLI
// parity test (tests/test_cli.py).  Writes <dir>/cli_<case>.{rules,jsonl}.
#include <cstdio>
#include <fstream>
#include <string>

#include "logtrawl/jsonl.hpp"
#include "logtrawl/loggen.hpp"
#include "logtrawl/pipeline.hpp"

using namespace logtrawl;

static void put(const std::string& path, const std::string& s) {
  std::ofstream(path, std::ios::binary) << s;
}

static void emit(const std::string& dir, const std::string& name, const std::string& rules_text,
                 const std::string& file, const std::string& text, const char* engine) {
  RuleSet rules = parse_rules(rules_text);
  EngineConfig cfg;
  cfg.engine = *engine_from_name(engine);
  LineIndex lines(text);
  put(dir + "/cli_" + name + ".rules", rules_text);
  put(dir + "/cli_" + name + "_" + engine + ".jsonl", render_alerts_jsonl(file, run_engine_scan(text, rules, cfg, &lines)));
}

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : ".";
  const char* engines[] = {"pfac_compact", "pfac_dense", "kmp", "ac_chunked"};
  // the reference's own CLI contract case (tests/cli_test.sh:20-33)
  for (const char* e : engines) emit(dir, "hit", "his-rule : HIS\nshe-rule : SHE\n", "hit.log", "SHIS\n", e);
  // escapes in names, bytes via \xNN, a generated corpus (generate_log seed 42)
  GenSpec spec;
  spec.size = 200000;
  spec.seed = 42;
  const std::string big = generate_log(spec).bytes;
  std::string rules_text = "q\"uote\\name : ab\ntab\tname : \\x41\\x42\n";
  const RuleSet rnd = random_rules(40, 3, 7);
  for (const Pattern& p : rnd.patterns) {
    std::string esc;
    for (unsigned char c : p.bytes) {
      char buf[8];
      std::snprintf(buf, sizeof buf, "\\x%02x", c);
      esc += buf;
    }
    rules_text += p.name + " : " + esc + "\n";
  }
  for (const char* e : engines) emit(dir, "big", rules_text, "big.log", big, e);
  return 0;
}
