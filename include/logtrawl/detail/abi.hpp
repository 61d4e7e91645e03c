#pragma once
// Glue between the drop-in C++ API and the C ABI (include/glop.h): one
// process-wide context per device and the mapping of glop_status codes onto
// the exception types the reference throws.
#include <cstdlib>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>

#include "glop.h"
#include "logtrawl/automaton.hpp"

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

}  // namespace logtrawl::detail

namespace logtrawl {
inline detail::DeviceTrieCache::~DeviceTrieCache() {
  if (trie) glop_trie_destroy(trie);
}
}  // namespace logtrawl
