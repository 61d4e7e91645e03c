// engine_capi.cpp -- libglop_engine.so: the drop-in C++ API (include/logtrawl,
// the reference's run_engine_scan, pipeline.hpp:49-100) behind a C ABI, for
// callers that reach the reference's engine through an FFI (ctypes, cgo, JNI)
// and for bench.py's `e2e_dropin` leg, which times exactly the call a
// reference C++ caller makes: run_engine_scan on a pageable host buffer.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "glop.h"
#include "logtrawl/pipeline.hpp"

namespace {
thread_local std::string g_engine_err;
}

extern "C" {

// A RuleSet: pattern i = bytes[off[i], off[i+1]), id i, name "r<i>".
void* glop_engine_rules_create(const uint8_t* bytes, const uint64_t* off, uint32_t k) {
  auto* r = new (std::nothrow) logtrawl::RuleSet();
  if (!r) return nullptr;
  for (uint32_t i = 0; i < k; ++i) {
    logtrawl::Pattern p;
    p.id = i;
    p.name = "r" + std::to_string(i);
    p.bytes.assign(reinterpret_cast<const char*>(bytes) + off[i], off[i + 1] - off[i]);
    r->max_len = std::max(r->max_len, p.bytes.size());
    r->patterns.push_back(std::move(p));
  }
  return r;
}

void glop_engine_rules_destroy(void* rules) { delete static_cast<logtrawl::RuleSet*>(rules); }

const char* glop_engine_last_error(void) { return g_engine_err.c_str(); }

// run_engine_scan(text, rules, {engine, prefix_len, workers, chunk_size},
// with_lines ? &LineIndex(text) : nullptr).  engine: 0 kmp, 1 pfac_dense,
// 2 pfac_compact, 3 ac_chunked.  Alerts as glop_alert records (+ lines when
// with_lines), library-owned (glop_free).  Returns 0, or 1 invalid_argument,
// 2 CapacityError, 3 logic_error, 4 other (glop_engine_last_error()).
int glop_engine_run(void* rules, const char* text, uint64_t n, int engine, uint64_t prefix_len, uint64_t chunk_size,
                    int with_lines, glop_alert** alerts, uint64_t** lines, uint64_t* n_alerts, uint64_t* stage1_hits) {
  try {
    logtrawl::EngineConfig cfg;
    cfg.engine = static_cast<logtrawl::EngineKind>(engine);
    cfg.prefix_len = prefix_len;
    if (chunk_size) cfg.chunk_size = chunk_size;
    const std::string_view tv(text, n);
    std::unique_ptr<logtrawl::LineIndex> idx;
    if (with_lines) idx = std::make_unique<logtrawl::LineIndex>(tv);
    const auto t0 = std::chrono::steady_clock::now();
    const logtrawl::ScanReport rep =
        logtrawl::run_engine_scan(tv, *static_cast<logtrawl::RuleSet*>(rules), cfg, idx.get());
    const auto t1 = std::chrono::steady_clock::now();
    const size_t na = rep.alerts.size();
    auto* a = static_cast<glop_alert*>(malloc(std::max<size_t>(na, 1) * sizeof(glop_alert)));
    auto* l = with_lines ? static_cast<uint64_t*>(malloc(std::max<size_t>(na, 1) * 8)) : nullptr;
    logtrawl::detail::parallel_for(na, [&](size_t lo, size_t hi) {
      for (size_t i = lo; i < hi; ++i) {
        a[i] = glop_alert{rep.alerts[i].offset, rep.alerts[i].rule_id, rep.alerts[i].pattern_len};
        if (l) l[i] = rep.alerts[i].line;
      }
    });
    if (std::getenv("GLOP_ENGINE_TIMING"))
      std::fprintf(stderr, "engine: run_engine_scan %.1f ms, to C records %.1f ms\n",
                   std::chrono::duration<double, std::milli>(t1 - t0).count(),
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count());
    *alerts = a;
    if (lines) *lines = l;
    *n_alerts = na;
    if (stage1_hits) *stage1_hits = rep.stage1_hits;
    return 0;
  } catch (const logtrawl::CapacityError& e) {
    g_engine_err = e.what();
    return 2;
  } catch (const std::invalid_argument& e) {
    g_engine_err = e.what();
    return 1;
  } catch (const std::logic_error& e) {
    g_engine_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_engine_err = e.what();
    return 4;
  }
}

}  // extern "C"
