// glop.cu -- host side of libglop.so: the C ABI declared in include/glop.h.
//
// Owns device memory, streams and kernel launches; flattens the reference's
// dense failureless trie (automaton.hpp:51-141) into the device layout once
// per automaton; orchestrates scan -> per-tile order -> gather, verification
// and KMP.  No CPU fallback: every matching computation runs on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <memory>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "glop.h"
#include "glop_kernels.cuh"
#include "pfac8.cuh"
#include "kmp.cuh"
#include "lines.cuh"
#include "pipeline.cuh"
#include "logtrawl/automaton.hpp"
#include "logtrawl/detail/abi.hpp"
#include "workload.hpp"

namespace glop {
// hostcopy.cpp: pageable -> pinned staging copy on a persistent host thread pool
void parallel_memcpy(void* dst, const void* src, size_t bytes);
}  // namespace glop
using namespace glop;

static_assert(sizeof(glop_hit) == 16, "glop_hit must match logtrawl::Hit");
static_assert(sizeof(DevHit) == sizeof(glop_hit), "device hit layout");
static_assert(sizeof(DevAlert) == sizeof(glop_alert), "device alert layout");

namespace {

thread_local std::string g_err;

glop_status fail(glop_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CU(expr)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(e_ == cudaErrorMemoryAllocation ? GLOP_ENOMEM : GLOP_ECUDA,            \
                  std::string(#expr) + ": " + cudaGetErrorString(e_));                   \
  } while (0)

#define TRY(expr)                          \
  do {                                     \
    glop_status s_ = (expr);               \
    if (s_ != GLOP_OK) return s_;          \
  } while (0)

// Growable device buffer.
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  glop_status ensure(size_t want) {
    if (want <= bytes) return GLOP_OK;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    size_t b = std::max<size_t>(want, 256);
    CU(cudaMalloc(&p, b));
    bytes = b;
    return GLOP_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Results of a text processed window by window (the streamed host pipeline,
// glop_stream_*): alerts and line numbers appended in text order, per-pattern
// counts and the LF count of the windows so far on the device.
struct Accum {
  DBuf alerts, lines, cnt;  // cnt: counts[k+1] | window counts[k+1] | lf
  uint64_t total = 0, hits = 0;
  uint32_t k = 0;
  bool want_lines = false;
  uint64_t* d_counts() { return cnt.as<uint64_t>(); }
  uint64_t* d_window_counts() { return cnt.as<uint64_t>() + k + 1; }
  uint64_t* d_lf() { return cnt.as<uint64_t>() + 2 * (k + 1); }
  void release() {
    alerts.release();
    lines.release();
    cnt.release();
  }
};

}  // namespace

struct glop_ctx {
  int device = 0;
  int num_sms = 148;
  size_t smem_optin = 0;
  cudaStream_t stream = nullptr;
  DBuf text, staging, out, dir, prefix, misc, keys, keys_alt, cub_tmp;
  DBuf keep, bcounts, bprefix, alerts, kmp_dfa, spill;
  DBuf sbuf[2];                                  // streamed text chunks (host-text pipeline)
  DBuf lcount, lprefix, loffs;                   // device LineIndex
  DBuf kcounts, keep8, counts_tmp;  // fused pipeline (pipeline.cuh)
  DBuf palerts, plines;                          // alerts (+ lines) of the host-facing pipeline calls
  std::string kmp_key;                           // pattern + failure table of the DFA in kmp_dfa
  Accum acc;                                     // streamed pipeline results
  cudaStream_t cstream = nullptr;                // H2D copies of the streamed pipeline
  void* pin[3] = {nullptr, nullptr, nullptr};    // pinned staging of pageable host text (ring)
  size_t pin_bytes = 0;                          // size of each pin[] buffer
  cudaEvent_t ev_pin[3] = {};                    // DMA out of pin[b] done
  cudaEvent_t ev_copied[2] = {}, ev_free[2] = {};
  unsigned long long* h_misc = nullptr;  // pinned readback
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;  // around the last scan kernel
  bool timed = false;
  uint64_t launches = 0;
  uint64_t fallbacks = 0;  // scans that took the exact global-key fallback
  std::mutex mu;
};

struct glop_trie {
  int device = 0;
  void* mem = nullptr;
  DevTrie view{};
  glop_trie_info info{};
  bool empty = true;      // no outputs: every scan is empty
  bool u16 = true;
  bool smem_filter = false, smem_direct = false, smem_jump = false;
  bool p8 = false;  // every output at depth >= 8: pfac8_kernel applies
  int p8_l1 = 0;  // pfac8 level-1/2 layout (kL1, see pfac8.cuh)
  mutable bool p8_careful = false;  // kCareful pfac8 kernel (set at upload; sticky after a fallback)
  uint32_t p8_lane_emits = 0;       // most hits one start position can emit
  uint32_t max_pid = 0;
};

struct glop_rules {
  int device = 0;
  void* mem = nullptr;
  DevRules view{};
  uint64_t max_len = 0;
};

namespace {

constexpr size_t kSmemMax = 232448;  // 227 KB opt-in per CTA on sm_100
constexpr uint64_t kStreamChunk = 256ull << 20;  // host-text pipeline chunk

struct Dev {
  explicit Dev(int d) { cudaGetDevice(&prev); if (prev != d) cudaSetDevice(d); dev = d; }
  ~Dev() { if (prev != dev) cudaSetDevice(prev); }
  int prev = 0, dev = 0;
};

size_t up16(size_t x) { return (x + 15) & ~size_t(15); }

glop_status sync_read(glop_ctx* c, const void* d_src, size_t bytes) {
  CU(cudaMemcpyAsync(c->h_misc, d_src, bytes, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return GLOP_OK;
}

// -------------------------------------------------------------- kernel launch
template <typename K>
glop_status launch_timed(glop_ctx* c, K k, int grid, const DevTrie& tr, const WarpScanParams& p,
                         const PfacLayout& L) {
  CU(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
  CU(cudaEventRecord(c->ev0, c->stream));
  k<<<grid, kWarpKernelThreads, L.total, c->stream>>>(tr, p, L);
  CU(cudaGetLastError());
  CU(cudaEventRecord(c->ev1, c->stream));
  c->timed = true;
  ++c->launches;
  return GLOP_OK;
}

template <typename E, uint32_t kS>
glop_status launch_pfac_s(glop_ctx* c, const glop_trie* t, const WarpScanParams& p, int grid) {
  const DevTrie& tr = t->view;
  const bool sh = t->smem_jump, st = t->smem_filter;
  const PfacLayout L = make_warp_layout(true, sh ? tr.jump_bytes : 0, st ? tr.table_bytes : 0);
  if (sh) return st ? launch_timed(c, pfac_warp_kernel<true, true, true, E, kS>, grid, tr, p, L)
                    : launch_timed(c, pfac_warp_kernel<true, false, true, E, kS>, grid, tr, p, L);
  return st ? launch_timed(c, pfac_warp_kernel<true, true, false, E, kS>, grid, tr, p, L)
            : launch_timed(c, pfac_warp_kernel<true, false, false, E, kS>, grid, tr, p, L);
}

template <typename E>
glop_status launch_pfac_e(glop_ctx* c, const glop_trie* t, bool filter, const WarpScanParams& p, int grid) {
  const DevTrie& tr = t->view;
  if (!filter) {
    const bool st = t->smem_direct;
    const PfacLayout L = make_warp_layout(false, 0, st ? tr.table_bytes : 0);
    return st ? launch_timed(c, pfac_warp_kernel<false, true, false, E, 0>, grid, tr, p, L)
              : launch_timed(c, pfac_warp_kernel<false, false, false, E, 0>, grid, tr, p, L);
  }
  if (tr.q == 4 && tr.stride == 5) return launch_pfac_s<E, 5>(c, t, p, grid);
  return launch_pfac_s<E, 0>(c, t, p, grid);
}

glop_status launch_pfac(glop_ctx* c, const glop_trie* t, bool filter, const WarpScanParams& p, int grid) {
  return t->u16 ? launch_pfac_e<uint16_t>(c, t, filter, p, grid) : launch_pfac_e<uint32_t>(c, t, filter, p, grid);
}

glop_status radix_sort_keys(glop_ctx* c, unsigned long long* in, unsigned long long* out,
                            unsigned long long n) {
  size_t tmp = 0;
  CU(cub::DeviceRadixSort::SortKeys(nullptr, tmp, in, out, n, 0, 64, c->stream));
  TRY(c->cub_tmp.ensure(tmp));
  CU(cub::DeviceRadixSort::SortKeys(c->cub_tmp.p, tmp, in, out, n, 0, 64, c->stream));
  return GLOP_OK;
}

// pfac8 launch geometry: one CTA per SM, kP8Warps contiguous warp segments
// per CTA, one staging region per warp.
struct P8Geom {
  uint32_t num_tiles, per, sub;
  int grid;
  unsigned long long regions, region;
};

glop_status p8_geometry(glop_ctx* c, const uint8_t* d_text, uint64_t own, P8Geom* G) {
  const uint32_t a = (uint32_t)((uintptr_t)d_text & 15);
  G->num_tiles = (uint32_t)((own + a + kP8Tile - 1) / kP8Tile);
  G->grid = (int)std::min<uint32_t>((G->num_tiles + kP8Warps - 1) / kP8Warps, (uint32_t)c->num_sms);
  G->per = (G->num_tiles + G->grid - 1) / G->grid;
  G->sub = (G->per + kP8Warps - 1) / kP8Warps;
  G->regions = (unsigned long long)G->grid * kP8Warps;
  TRY(c->bcounts.ensure(8 * G->regions));
  TRY(c->misc.ensure(64));
  unsigned long long region =
      std::max<unsigned long long>(256, (std::max<uint64_t>(1 << 20, own / 512) + G->regions - 1) / G->regions);
  if (c->staging.bytes < region * G->regions * sizeof(glop_hit))
    TRY(c->staging.ensure(region * G->regions * sizeof(glop_hit)));
  G->region = c->staging.bytes / sizeof(glop_hit) / G->regions;
  return GLOP_OK;
}

glop_status launch_pfac8(glop_ctx* c, const glop_trie* t, const P8Geom& G, const P8Params& p) {
  using KF = void (*)(const DevTrie, const P8Params, const P8Layout);
#define GLOP_P8_K(w, l, c) {pfac8_kernel<w, l, uint16_t, c>, pfac8_kernel<w, l, uint32_t, c>}
#define GLOP_P8_L(w, c) \
  GLOP_P8_K(w, 0, c), GLOP_P8_K(w, 1, c), GLOP_P8_K(w, 2, c), GLOP_P8_K(w, 3, c), GLOP_P8_K(w, 4, c), \
      GLOP_P8_K(w, 5, c)
  static const KF table[2][2][6][2] = {{{GLOP_P8_L(false, false)}, {GLOP_P8_L(true, false)}},
                                       {{GLOP_P8_L(false, true)}, {GLOP_P8_L(true, true)}}};
#undef GLOP_P8_L
#undef GLOP_P8_K
  const P8Layout L = make_p8_layout();
  const KF k = table[t->p8_careful][t->info.max_depth > 8][t->p8_l1][t->u16 ? 0 : 1];
  CU(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
  CU(cudaEventRecord(c->ev0, c->stream));
  k<<<G.grid, kP8Threads, L.total, c->stream>>>(t->view, p, L);
  CU(cudaGetLastError());
  CU(cudaEventRecord(c->ev1, c->stream));
  c->timed = true;
  ++c->launches;
  return GLOP_OK;
}

P8Params p8_params(glop_ctx* c, const glop_trie* t, const P8Geom& G, const uint8_t* d_text, uint64_t n, uint64_t own,
                   uint64_t base) {
  P8Params p{};
  p.text = d_text;
  p.n = n;
  p.own = own;
  p.base = base;
  p.num_tiles = G.num_tiles;
  p.per = G.per;
  p.sub = G.sub;
  p.mode = 0;
  p.staging = reinterpret_cast<DevHit*>(c->staging.p);
  p.region = G.region;
  p.counts = c->bcounts.as<unsigned long long>();
  p.g_count = c->misc.as<unsigned long long>();
  p.dmask8 = t->view.dmask8;
  return p;
}

// pfac8 path (every output at depth >= 8), same contract as below.
glop_status pfac8_scan_impl(glop_ctx* c, const glop_trie* t, const uint8_t* d_text, uint64_t n,
                            uint64_t own, uint64_t base, glop_hit* d_out, uint64_t cap, uint64_t* n_hits) {
  P8Geom G;
  TRY(p8_geometry(c, d_text, own, &G));
  auto* g = c->misc.as<unsigned long long>();
  for (int attempt = 0; attempt < 3; ++attempt) {
    CU(cudaMemsetAsync(c->misc.p, 0, 64, c->stream));
    P8Params p = p8_params(c, t, G, d_text, n, own, base);
    TRY(launch_pfac8(c, t, G, p));
    // ordered output, enqueued before the flags are known (see gather_regions_kernel)
    ++c->launches;
    gather_regions_kernel<DevHit><<<(uint32_t)std::min<unsigned long long>(G.regions, 2ull * c->num_sms), 256, 0,
                                    c->stream>>>(c->bcounts.as<unsigned long long>(), (uint32_t)G.regions, G.region,
                                                 reinterpret_cast<const DevHit*>(c->staging.p),
                                                 reinterpret_cast<DevHit*>(d_out), cap);
    CU(cudaGetLastError());
    TRY(sync_read(c, c->misc.p, 32));
    const unsigned long long total = c->h_misc[kStTotal], maxregion = c->h_misc[kStMaxRegion];
    const unsigned flags = (unsigned)(c->h_misc[kStFlags] & 0xffffffffu);
    if (getenv("GLOP_DEBUG"))
      fprintf(stderr, "pfac8: tiles %u grid %d per %u sub %u region %llu -> total %llu flags %u maxregion %llu\n",
              G.num_tiles, G.grid, G.per, G.sub, G.region, total, flags, maxregion);
    *n_hits = total;
    if (flags & 1u) {
      ++c->fallbacks;
      t->p8_careful = true;  // later scans of this automaton replay lanes from an empty buffer
      // one lane of a drain round produced more hits than the warp's buffer
      // holds: exact fallback -- global keys, device radix sort.  A counting
      // pass (keys_cap = 0) sizes the key buffer.
      CU(cudaMemsetAsync(c->misc.p, 0, 64, c->stream));
      p.mode = 1;
      p.keys = nullptr;
      p.keys_cap = 0;
      TRY(launch_pfac8(c, t, G, p));
      TRY(sync_read(c, c->misc.p, 32));
      const unsigned long long exact_total = c->h_misc[kStKeys];
      *n_hits = exact_total;
      if (exact_total > cap) return fail(GLOP_ECAPACITY, "pfac_scan: output capacity");
      TRY(c->keys.ensure(exact_total * 8 + 8));
      TRY(c->keys_alt.ensure(exact_total * 8 + 8));
      CU(cudaMemsetAsync(c->misc.p, 0, 64, c->stream));
      p.keys = c->keys.as<unsigned long long>();
      p.keys_cap = exact_total;
      TRY(launch_pfac8(c, t, G, p));
      if (exact_total == 0) return GLOP_OK;
      TRY(radix_sort_keys(c, c->keys.as<unsigned long long>(), c->keys_alt.as<unsigned long long>(), exact_total));
      c->launches += 2;
      keys_to_hits_kernel<<<std::max<unsigned long long>(1, std::min<unsigned long long>((exact_total + 255) / 256, 4096)),
                            256, 0, c->stream>>>(c->keys_alt.as<unsigned long long>(), exact_total, t->view.pid_len,
                                                 reinterpret_cast<DevHit*>(d_out));
      CU(cudaGetLastError());
      CU(cudaStreamSynchronize(c->stream));
      return GLOP_OK;
    }
    if (maxregion > G.region) {  // a warp's staging region overflowed: grow, rerun
      const unsigned long long region = maxregion + maxregion / 4 + 64;
      c->staging.release();
      TRY(c->staging.ensure(region * G.regions * sizeof(glop_hit)));
      G.region = region;
      continue;
    }
    if (total > cap) return fail(GLOP_ECAPACITY, "pfac_scan: output capacity");
    return GLOP_OK;
  }
  (void)g;
  return fail(GLOP_ECUDA, "pfac_scan: staging did not converge");
}

// PFAC over d_text[0, n): starts [0, own), offsets + base, sorted hits to out.
glop_status pfac_scan_device_impl(glop_ctx* c, const glop_trie* t, const uint8_t* d_text,
                                  uint64_t n, uint64_t own, uint64_t base, glop_pfac_kernel kind,
                                  glop_hit* d_out, uint64_t cap, uint64_t* n_hits) {
  *n_hits = 0;
  if (own > n) return fail(GLOP_EINVAL, "pfac_scan: own > n");
  if (own == 0 || t->empty) return GLOP_OK;
  if (kind == GLOP_PFAC_PREFIX8 && !t->p8)
    return fail(GLOP_EINVAL, "pfac_scan: PREFIX8 kernel needs every output at depth >= 8");
  // pfac8 keys are (offset << 24 | id): offsets < 2^40, ids < 2^24
  const bool p8_ok = t->p8 && t->max_pid < (1u << 24) && base + n < (1ull << 40);
  if (kind == GLOP_PFAC_PREFIX8 && !p8_ok)
    return fail(GLOP_EINVAL, "pfac_scan: PREFIX8 kernel needs ids < 2^24 and offsets < 2^40");
  if ((kind == GLOP_PFAC_AUTO && p8_ok) || kind == GLOP_PFAC_PREFIX8)
    return pfac8_scan_impl(c, t, d_text, n, own, base, d_out, cap, n_hits);
  const bool filter = kind != GLOP_PFAC_DIRECT;
  // tiles are aligned to the 16-byte granule holding the text start
  const uint32_t num_tiles = (uint32_t)((own + ((uintptr_t)d_text & 15) + kTile - 1) / kTile);
  const unsigned long long nseg = num_tiles;
  const uint32_t nb = (uint32_t)((nseg + kSegPerBlock - 1) / kSegPerBlock);
  const int grid = (int)std::min<uint32_t>(num_tiles, (uint32_t)c->num_sms);
  const unsigned long long regions = (unsigned long long)grid * kConsumerWarps;
  TRY(c->dir.ensure(sizeof(SegDir) * nseg));
  TRY(c->bcounts.ensure(4ull * nb));
  TRY(c->prefix.ensure(8ull * nb + 8));
  TRY(c->misc.ensure(64));
  unsigned long long region = std::max<unsigned long long>(64, (std::max<uint64_t>(1 << 20, own / 512) + regions - 1) / regions);
  if (c->staging.bytes < region * regions * sizeof(glop_hit))
    TRY(c->staging.ensure(region * regions * sizeof(glop_hit)));
  region = c->staging.bytes / sizeof(glop_hit) / regions;
  auto* g = c->misc.as<unsigned long long>();

  for (int attempt = 0; attempt < 3; ++attempt) {
    CU(cudaMemsetAsync(c->misc.p, 0, 32, c->stream));
    WarpScanParams p{};
    p.text = d_text;
    p.n = n;
    p.own = own;
    p.base = base;
    p.num_tiles = num_tiles;
    p.mode = 0;
    p.staging = reinterpret_cast<DevHit*>(c->staging.p);
    p.region = region;
    p.dir = c->dir.as<SegDir>();
    p.g_count = g;
    TRY(launch_pfac(c, t, filter, p, grid));
    TRY(sync_read(c, c->misc.p, 32));
    const unsigned long long total = c->h_misc[0], maxregion = c->h_misc[2];
    const unsigned flags = (unsigned)(c->h_misc[1] & 0xffffffffu);
    *n_hits = total;
    if (flags & 1u) {
      ++c->fallbacks;
      // a slice produced more hits than its shared-memory buffer holds:
      // exact fallback -- global keys, device radix sort
      if (t->max_pid >= (1u << 24) || base + n >= (1ull << 40))
        return fail(GLOP_ECAPACITY, "pfac_scan: hit density fallback limited to 2^24 ids / 2^40 bytes");
      if (total > cap) return fail(GLOP_ECAPACITY, "pfac_scan: output capacity");
      TRY(c->keys.ensure(total * 8));
      TRY(c->keys_alt.ensure(total * 8));
      CU(cudaMemsetAsync(c->misc.p, 0, 32, c->stream));
      p.mode = 1;
      p.keys = c->keys.as<unsigned long long>();
      p.keys_cap = total;
      TRY(launch_pfac(c, t, filter, p, grid));
      TRY(radix_sort_keys(c, c->keys.as<unsigned long long>(), c->keys_alt.as<unsigned long long>(), total));
      c->launches += 2;
      keys_to_hits_kernel<<<std::max<unsigned long long>(1, std::min<unsigned long long>((total + 255) / 256, 4096)), 256, 0,
                            c->stream>>>(c->keys_alt.as<unsigned long long>(), total, t->view.pid_len,
                                         reinterpret_cast<DevHit*>(d_out));
      CU(cudaGetLastError());
      CU(cudaStreamSynchronize(c->stream));
      return GLOP_OK;
    }
    if (maxregion > region) {  // a warp's staging region overflowed: grow, rerun
      region = maxregion + maxregion / 4 + 64;
      c->staging.release();
      TRY(c->staging.ensure(region * regions * sizeof(glop_hit)));
      continue;
    }
    if (total > cap) return fail(GLOP_ECAPACITY, "pfac_scan: output capacity");
    if (total == 0) return GLOP_OK;
    c->launches += 3;
    seg_reduce_kernel<<<nb, 1024, 0, c->stream>>>(c->dir.as<SegDir>(), nseg, c->bcounts.as<uint32_t>());
    block_prefix_kernel<<<1, 1024, 0, c->stream>>>(c->bcounts.as<uint32_t>(), nb, c->prefix.as<unsigned long long>(),
                                                   c->prefix.as<unsigned long long>() + nb);
    seg_gather_kernel<DevHit><<<nb, 1024, 0, c->stream>>>(c->dir.as<SegDir>(), nseg, c->prefix.as<unsigned long long>(),
                                                          (uint32_t)grid, region,
                                                          reinterpret_cast<const DevHit*>(c->staging.p),
                                                          reinterpret_cast<DevHit*>(d_out));
    CU(cudaGetLastError());
    return GLOP_OK;
  }
  return fail(GLOP_ECUDA, "pfac_scan: staging did not converge");
}

// KMP DFA (see kmp.cuh): replays kmp.hpp:52-66 for each (state, byte):
// next state | match << 13 | comparisons << 14.
void build_kmp_dfa(const uint8_t* p, uint32_t m, const uint32_t* fail_tab, std::vector<uint32_t>& dfa) {
  dfa.assign((size_t)m * 256, 0);
  for (uint32_t j0 = 0; j0 < m; ++j0)
    for (uint32_t b = 0; b < 256; ++b) {
      uint32_t j = j0, cmp = 0, match = 0;
      for (;;) {
        ++cmp;
        if (b == p[j]) {
          ++j;
          if (j == m) {
            match = 1;
            j = fail_tab[m - 1];
          }
          break;
        } else if (j > 0) {
          j = fail_tab[j - 1];
        } else {
          break;
        }
      }
      dfa[(size_t)j0 * 256 + b] = j | (match << 13) | (cmp << 14);
    }
}

glop_status kmp_seq_impl(glop_ctx* c, const uint8_t* pat, uint32_t m, const uint32_t* fail_tab, const uint8_t* d_text,
                         uint64_t n, uint64_t* d_out, uint64_t cap, uint64_t* n_offsets, uint64_t* comparisons);

// KMP over d_text = global [base, base + n): starts in [skip, own) (local) are
// reported as base + start, and the comparisons the sequential scan makes at
// positions [skip, own) are added -- exact when skip is 0 (the text's true
// start) or >= m - 1 (a left context long enough to recover the state).
glop_status kmp_device_impl(glop_ctx* c, const uint8_t* pat, uint32_t m, const uint32_t* fail_tab,
                            const uint8_t* d_text, uint64_t n, uint64_t own, uint64_t base,
                            uint64_t* d_out, uint64_t cap, uint64_t* n_offsets,
                            uint64_t* comparisons, uint64_t skip = 0, glop_pipeline_ticket* ticket = nullptr) {
  *n_offsets = 0;
  if (own > n || skip > own) return fail(GLOP_EINVAL, "kmp_search: own > n or skip > own");
  if (m == 0 || n < m || own == skip) return GLOP_OK;  // kmp.hpp:50
  // chunks resynchronise from the previous m-1 bytes, which is exact for the
  // pattern's own prefix function (kmp.hpp:25-36); any other table (or a
  // pattern too long for the DFA) runs the sequential walk, whole texts only
  bool canonical = m < 8192;
  for (uint32_t i = 0, k = 0; i < m && canonical; ++i) {
    if (i > 0) {
      while (k > 0 && pat[i] != pat[k]) k = fail_tab[k - 1];
      if (pat[i] == pat[k]) ++k;
    }
    canonical = fail_tab[i] == (i ? k : 0u);
  }
  if (!canonical) {
    if (own != n || base != 0 || skip != 0)
      return fail(GLOP_EINVAL, "kmp_search: shards need the pattern's own prefix function and m < 8192");
    return kmp_seq_impl(c, pat, m, fail_tab, d_text, n, d_out, cap, n_offsets, comparisons);
  }
  // the DFA of the context's last pattern stays on the device
  std::string key(reinterpret_cast<const char*>(pat), m);
  key.append(reinterpret_cast<const char*>(fail_tab), (size_t)m * 4);
  if (key != c->kmp_key) {
    std::vector<uint32_t> dfa;
    build_kmp_dfa(pat, m, fail_tab, dfa);
    TRY(c->kmp_dfa.ensure(dfa.size() * 4));
    // (stream-ordered after the kernels reading the previous DFA; a pageable
    // source is staged before the call returns)
    CU(cudaMemcpyAsync(c->kmp_dfa.p, dfa.data(), dfa.size() * 4, cudaMemcpyHostToDevice, c->stream));
    c->kmp_key.swap(key);
  }
  const uint64_t end_lim = std::min<uint64_t>(own + m - 1, n);  // starts < own
  const uint32_t a = (uint32_t)((uintptr_t)d_text & 15);
  const uint32_t num_tiles = (uint32_t)((end_lim + a + kK3Tile - 1) / kK3Tile);
  const int grid = (int)std::min<uint32_t>((num_tiles + kK3Warps - 1) / kK3Warps, (uint32_t)c->num_sms);
  const uint32_t per = (num_tiles + grid - 1) / grid, sub = (per + kK3Warps - 1) / kK3Warps;
  const unsigned long long regions = (unsigned long long)grid * kK3Warps;
  TRY(c->bcounts.ensure(8 * regions));
  TRY(c->misc.ensure(64));
  unsigned long long region = std::max<unsigned long long>(256, (own / 8192 + regions - 1) / regions);
  if (c->staging.bytes < region * regions * 8) TRY(c->staging.ensure(region * regions * 8));
  region = c->staging.bytes / 8 / regions;
  auto* g = c->misc.as<unsigned long long>();
  const bool smem_dfa = m <= kK3SmemDfaMax;
  const K3Layout L = make_k3_layout(m, smem_dfa);
  auto launch = [&](const K3Params& p) -> glop_status {
    auto k = smem_dfa ? kmp3_kernel<true> : kmp3_kernel<false>;
    CU(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
    CU(cudaEventRecord(c->ev0, c->stream));
    k<<<grid, kK3Threads, L.total, c->stream>>>(p, L);
    CU(cudaGetLastError());
    CU(cudaEventRecord(c->ev1, c->stream));
    c->timed = true;
    ++c->launches;
    return GLOP_OK;
  };
  for (int attempt = 0; attempt < 3; ++attempt) {
    CU(cudaMemsetAsync(c->misc.p, 0, 32, c->stream));
    K3Params p{};
    p.text = d_text;
    p.n = n;
    p.own = own;
    p.end_lim = end_lim;
    p.base = base;
    p.skip = skip;
    p.m = m;
    p.p0 = pat[0];
    p.num_tiles = num_tiles;
    p.per = per;
    p.sub = sub;
    p.dfa = c->kmp_dfa.as<uint32_t>();
    p.staging = c->staging.as<unsigned long long>();
    p.region = region;
    p.counts = c->bcounts.as<unsigned long long>();
    p.g_count = g;
    p.comparisons = g + 2;
    TRY(launch(p));
    // ordered output, enqueued before the flags are known (see gather_regions_kernel)
    ++c->launches;
    gather_regions_kernel<unsigned long long>
        <<<(uint32_t)std::min<unsigned long long>(regions, 2ull * c->num_sms), 256, 0, c->stream>>>(
            c->bcounts.as<unsigned long long>(), (uint32_t)regions, region, c->staging.as<unsigned long long>(),
            reinterpret_cast<unsigned long long*>(d_out), cap);
    CU(cudaGetLastError());
    if (ticket) {  // no host wait: the status block lands in the ticket
      ticket->region = region;
      ticket->hit_cap = cap;
      ticket->alert_cap = 0;
      ticket->stage2 = 3;  // (KMP ticket)
      ticket->done = 0;
      CU(cudaMemcpyAsync(ticket->raw, c->misc.p, sizeof ticket->raw, cudaMemcpyDeviceToHost, c->stream));
      return GLOP_OK;
    }
    TRY(sync_read(c, c->misc.p, 32));
    const unsigned long long total = c->h_misc[0], maxregion = c->h_misc[3];
    const unsigned flags = (unsigned)(c->h_misc[1] & 0xffffffffu);
    *n_offsets = total;
    if (flags & 1u) {
      // > kK3Hits matches in one warp tile: exact fallback -- every match as a
      // global key, then a device radix sort.
      if (comparisons) *comparisons += c->h_misc[2];
      if (total > cap) return fail(GLOP_ECAPACITY, "kmp_search: output capacity");
      TRY(c->keys.ensure(total * 8 + 8));
      CU(cudaMemsetAsync(c->misc.p, 0, 32, c->stream));
      p.mode = 1;
      p.keys = c->keys.as<unsigned long long>();
      p.keys_cap = total;
      TRY(launch(p));
      TRY(radix_sort_keys(c, c->keys.as<unsigned long long>(), reinterpret_cast<unsigned long long*>(d_out), total));
      CU(cudaStreamSynchronize(c->stream));
      return GLOP_OK;
    }
    if (maxregion > region) {  // a warp's staging region overflowed: grow, rerun
      region = maxregion + maxregion / 4 + 64;
      c->staging.release();
      TRY(c->staging.ensure(region * regions * 8));
      continue;
    }
    if (comparisons) *comparisons += c->h_misc[2];
    if (total > cap) return fail(GLOP_ECAPACITY, "kmp_search: output capacity");
    return GLOP_OK;
  }
  return fail(GLOP_ECUDA, "kmp_search: staging did not converge");
}

glop_status to_device_text(glop_ctx* c, const uint8_t* text, uint64_t n, int on_device,
                           const uint8_t** d_text) {
  if (on_device || n == 0) {
    *d_text = text;
    return GLOP_OK;
  }
  TRY(c->text.ensure(n + 64));
  CU(cudaMemcpyAsync(c->text.p, text, n, cudaMemcpyHostToDevice, c->stream));
  *d_text = c->text.as<uint8_t>();
  return GLOP_OK;
}

// Hits were not in (offset, id) order: order the alerts on the device, as the
// reference sorts them (verify.hpp:100-103).  end = largest global offset + 1.
glop_status sort_alerts(glop_ctx* c, const glop_rules* r, uint64_t end, glop_alert* d_out, uint64_t kept) {
  if (kept < 2) return GLOP_OK;
  if (r->view.n_patterns > (1u << 24) || end >= (1ull << 40))
    return fail(GLOP_EINVAL, "verify_hits: unsorted hits need ids < 2^24 and offsets < 2^40");
  TRY(c->keys.ensure(kept * 8));
  TRY(c->keys_alt.ensure(kept * 8));
  const uint32_t grid = (uint32_t)std::min<uint64_t>((kept + 255) / 256, 4096);
  c->launches += 2;
  alerts_to_keys_kernel<<<grid, 256, 0, c->stream>>>(reinterpret_cast<DevAlert*>(d_out), kept,
                                                     c->keys.as<unsigned long long>());
  TRY(radix_sort_keys(c, c->keys.as<unsigned long long>(), c->keys_alt.as<unsigned long long>(), kept));
  keys_to_alerts_kernel<<<grid, 256, 0, c->stream>>>(c->keys_alt.as<unsigned long long>(), kept, r->view,
                                                     reinterpret_cast<DevAlert*>(d_out));
  CU(cudaGetLastError());
  return GLOP_OK;
}

glop_status verify_device_impl(glop_ctx* c, const glop_rules* r, const uint8_t* d_text, uint64_t n,
                               uint64_t base, const glop_hit* d_hits, uint64_t n_hits, glop_alert* d_out,
                               uint64_t* n_alerts, uint64_t* d_counts) {
  *n_alerts = 0;
  if (n_hits == 0) return GLOP_OK;
  if (r->max_len <= r->view.prefix_len) {  // every hit is auto-verified: one pass
    TRY(c->misc.ensure(64));
    CU(cudaMemsetAsync(c->misc.p, 0, 16, c->stream));
    auto* fl_all = reinterpret_cast<unsigned int*>(c->misc.as<unsigned long long>() + 1);
    ++c->launches;
    verify_all_kernel<<<(uint32_t)std::min<uint64_t>((n_hits + 1023) / 1024, 2u * c->num_sms), 1024, 0, c->stream>>>(
        r->view, base, n, reinterpret_cast<const DevHit*>(d_hits), n_hits, reinterpret_cast<DevAlert*>(d_out),
        reinterpret_cast<unsigned long long*>(d_counts), fl_all);
    CU(cudaGetLastError());
    TRY(sync_read(c, c->misc.p, 16));
    const unsigned fl = (unsigned)(c->h_misc[1] & 0xffffffffu);
    if (fl & 1u) return fail(GLOP_ELOGIC, "verify_hits: hit extends past end of text");
    *n_alerts = n_hits;
    if (fl & 2u) return sort_alerts(c, r, base + n, d_out, n_hits);
    return GLOP_OK;
  }
  const uint32_t nb = (uint32_t)((n_hits + kVerifyBlock - 1) / kVerifyBlock);
  TRY(c->keep.ensure(n_hits));
  TRY(c->bcounts.ensure(nb * 4));
  TRY(c->bprefix.ensure(nb * 8 + 8));
  TRY(c->misc.ensure(64));
  CU(cudaMemsetAsync(c->misc.p, 0, 16, c->stream));
  auto* flags = reinterpret_cast<unsigned int*>(c->misc.as<unsigned long long>() + 1);
  auto* total = c->misc.as<unsigned long long>();
  c->launches += 2;
  verify_flags_kernel<<<nb, kVerifyBlock, 0, c->stream>>>(
      r->view, d_text, base, n, reinterpret_cast<const DevHit*>(d_hits), n_hits, c->keep.as<uint8_t>(),
      c->bcounts.as<uint32_t>(), flags);
  block_prefix_kernel<<<1, 1024, 0, c->stream>>>(c->bcounts.as<uint32_t>(), nb,
                                                 c->bprefix.as<unsigned long long>(), total);
  CU(cudaGetLastError());
  TRY(sync_read(c, c->misc.p, 16));
  const unsigned long long kept = c->h_misc[0];
  const unsigned fl = (unsigned)(c->h_misc[1] & 0xffffffffu);
  if (fl & 1u) return fail(GLOP_ELOGIC, "verify_hits: hit extends past end of text");
  ++c->launches;
  const bool hist = d_counts && r->view.n_patterns <= kHistBins;
  verify_scatter_kernel<<<nb, kVerifyBlock, 0, c->stream>>>(
      r->view, reinterpret_cast<const DevHit*>(d_hits), n_hits, c->keep.as<uint8_t>(),
      c->bprefix.as<unsigned long long>(), reinterpret_cast<DevAlert*>(d_out),
      hist ? nullptr : reinterpret_cast<unsigned long long*>(d_counts));
  if (hist && kept) {
    ++c->launches;
    alert_histogram_kernel<<<(uint32_t)std::min<uint64_t>((kept + 1023) / 1024, c->num_sms), 1024, 0, c->stream>>>(
        reinterpret_cast<const DevAlert*>(d_out), kept, r->view.n_patterns,
        reinterpret_cast<unsigned long long*>(d_counts));
  }
  CU(cudaGetLastError());
  *n_alerts = kept;
  if (fl & 2u) return sort_alerts(c, r, base + n, d_out, kept);
  return GLOP_OK;
}

// Device-resident scan + verify + counts (the device half of run_engine_scan's
// PFAC branch).  pfac8 automata take the fused path of pipeline.cuh: every
// kernel is enqueued back to back and the host reads one status block at the
// end.  A scan that needs the exact fallback or a larger staging region, and
// non-pfac8 automata, go through pfac_scan_device_impl + verify_device_impl.
// d_hits (optional) receives the ordered hits (hit_cap records); d_counts
// (optional) the per-pattern alert counts (overwritten, not accumulated).
glop_status pipeline_device_impl(glop_ctx* c, const glop_trie* t, const glop_rules* r, const uint8_t* d_text,
                                 uint64_t n, uint64_t own, uint64_t base, glop_hit* d_hits, uint64_t hit_cap,
                                 glop_alert* d_alerts, uint64_t alert_cap, uint64_t* d_counts, uint64_t* n_hits,
                                 uint64_t* n_alerts, glop_pipeline_ticket* ticket = nullptr) {
  *n_hits = *n_alerts = 0;
  if (own > n) return fail(GLOP_EINVAL, "run_pfac_pipeline: own > n");
  const uint32_t k = r->view.n_patterns;
  if (!d_counts) {
    TRY(c->counts_tmp.ensure((size_t)(k + 1) * 8));
    d_counts = c->counts_tmp.as<uint64_t>();
  }
  const bool fused = t->p8 && !t->empty && own > 0 && t->max_pid < (1u << 24) && base + n < (1ull << 40) &&
                     !getenv("GLOP_NO_FUSED");
  if (fused) {
    P8Geom G;
    TRY(p8_geometry(c, d_text, own, &G));
    const bool stage2 = r->max_len > r->view.prefix_len;
    if (stage2) {
      TRY(c->kcounts.ensure(8 * G.regions));
      TRY(c->keep8.ensure(G.regions * G.region));
    }
    auto* g = c->misc.as<unsigned long long>();
    CU(cudaMemsetAsync(c->misc.p, 0, 64, c->stream));
    P8Params p = p8_params(c, t, G, d_text, n, own, base);
    p.zero = reinterpret_cast<unsigned long long*>(d_counts);  // (the scan's grid zeroes the counts)
    p.nzero = k;
    TRY(launch_pfac8(c, t, G, p));
    const auto* cnt = c->bcounts.as<unsigned long long>();
    const uint32_t egrid = (uint32_t)std::min<unsigned long long>(G.regions, 2ull * c->num_sms);
    const uint32_t hist_bins = (size_t)k * 4 <= kSmemMax - 2048 ? k : 0;
    const size_t hist_bytes = (size_t)hist_bins * 4;
    if (stage2) {
      ++c->launches;
      p8_keep_kernel<<<(uint32_t)std::min<unsigned long long>(G.regions, 8ull * c->num_sms), 256, 0, c->stream>>>(
          r->view, d_text, base, n, cnt, (uint32_t)G.regions, G.region, reinterpret_cast<const DevHit*>(c->staging.p),
          c->keep8.as<uint8_t>(), c->kcounts.as<unsigned long long>(), g + kStVerify);
      CU(cudaFuncSetAttribute(p8_emit_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hist_bytes));
      p8_emit_kernel<true><<<egrid, 1024, hist_bytes, c->stream>>>(
          r->view, base, n, cnt, (uint32_t)G.regions, G.region, reinterpret_cast<const DevHit*>(c->staging.p),
          c->keep8.as<uint8_t>(), c->kcounts.as<unsigned long long>(), reinterpret_cast<DevHit*>(d_hits),
          d_hits ? hit_cap : 0, reinterpret_cast<DevAlert*>(d_alerts), alert_cap,
          reinterpret_cast<unsigned long long*>(d_counts), hist_bins, g);
    } else {
      CU(cudaFuncSetAttribute(p8_emit_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hist_bytes));
      p8_emit_kernel<false><<<egrid, 1024, hist_bytes, c->stream>>>(
          r->view, base, n, cnt, (uint32_t)G.regions, G.region, reinterpret_cast<const DevHit*>(c->staging.p),
          nullptr, nullptr, reinterpret_cast<DevHit*>(d_hits), d_hits ? hit_cap : 0,
          reinterpret_cast<DevAlert*>(d_alerts), alert_cap, reinterpret_cast<unsigned long long*>(d_counts),
          hist_bins, g);
    }
    ++c->launches;
    CU(cudaGetLastError());
    if (ticket) {  // no host wait: the status block lands in the ticket, read after the stream syncs
      ticket->region = G.region;
      ticket->hit_cap = d_hits ? hit_cap : ~0ull;
      ticket->alert_cap = alert_cap;
      ticket->stage2 = stage2;
      ticket->done = 0;
      CU(cudaMemcpyAsync(ticket->raw, c->misc.p, sizeof ticket->raw, cudaMemcpyDeviceToHost, c->stream));
      return GLOP_OK;
    }
    TRY(sync_read(c, c->misc.p, 64));
    const unsigned long long* h = c->h_misc;
    const unsigned flags = (unsigned)(h[kStFlags] & 0xffffffffu);
    if (!(flags & 1u) && h[kStMaxRegion] <= G.region) {
      if (h[kStVerify] & 1u) return fail(GLOP_ELOGIC, "verify_hits: hit extends past end of text");
      *n_hits = h[kStTotal];
      *n_alerts = stage2 ? h[kStKept] : h[kStTotal];
      if ((d_hits && *n_hits > hit_cap) || *n_alerts > alert_cap)
        return fail(GLOP_ECAPACITY, "run_pfac_pipeline: output capacity");
      return GLOP_OK;
    }
    // overflow: the general path below handles the exact fallback / regrowth
  }
  glop_hit* hits = d_hits;
  uint64_t cap = hit_cap;
  if (!hits) {
    cap = std::max<uint64_t>(1 << 16, c->out.bytes / sizeof(glop_hit));
    TRY(c->out.ensure(cap * sizeof(glop_hit)));
    hits = c->out.as<glop_hit>();
  }
  uint64_t nh = 0;
  glop_status s = pfac_scan_device_impl(c, t, d_text, n, own, base, GLOP_PFAC_AUTO, hits, cap, &nh);
  if (s == GLOP_ECAPACITY && !d_hits && nh > cap) {
    c->out.release();
    cap = nh;
    TRY(c->out.ensure(cap * sizeof(glop_hit)));
    hits = c->out.as<glop_hit>();
    s = pfac_scan_device_impl(c, t, d_text, n, own, base, GLOP_PFAC_AUTO, hits, cap, &nh);
  }
  *n_hits = nh;
  if (s != GLOP_OK) return s;
  if (nh > alert_cap) {  // alerts <= hits; only a short alert buffer can overflow
    TRY(c->alerts.ensure(nh * sizeof(glop_alert)));
    CU(cudaMemsetAsync(d_counts, 0, (size_t)k * 8, c->stream));
    uint64_t kept = 0;
    TRY(verify_device_impl(c, r, d_text, n, base, hits, nh, c->alerts.as<glop_alert>(), &kept, d_counts));
    *n_alerts = kept;
    if (kept > alert_cap) return fail(GLOP_ECAPACITY, "run_pfac_pipeline: output capacity");
    CU(cudaMemcpyAsync(d_alerts, c->alerts.p, kept * sizeof(glop_alert), cudaMemcpyDeviceToDevice, c->stream));
    return GLOP_OK;
  }
  CU(cudaMemsetAsync(d_counts, 0, (size_t)k * 8, c->stream));
  return verify_device_impl(c, r, d_text, n, base, hits, nh, d_alerts, n_alerts, d_counts);
}

// Host-text pipeline for large inputs (streaming ingest):
// the text is copied in kStreamChunk pieces (+ a halo for the trie walk and
// the stage-2 suffix compare) on a copy stream into two device buffers, so
// the H2D copy of chunk i+1 overlaps the scan + verify of chunk i.  Chunk
// results are exact and ordered (ownership of starts, scan.hpp:230-232), so
// the alerts are the concatenation of the chunks' alerts.
glop_status line_numbers_impl(glop_ctx* c, const uint8_t* d_text, uint64_t n, uint64_t base, const void* d_recs,
                              uint32_t stride, uint64_t count, uint64_t* d_lines, const uint64_t* d_line_base,
                              uint64_t* d_lf_acc);

// Grows a device buffer to `want` bytes keeping its first `keep` bytes.
glop_status grow_keep(glop_ctx* c, DBuf& b, size_t want, size_t keep) {
  if (want <= b.bytes) return GLOP_OK;
  DBuf bigger;
  TRY(bigger.ensure(std::max<size_t>(want, 2 * b.bytes)));
  if (keep) CU(cudaMemcpyAsync(bigger.p, b.p, keep, cudaMemcpyDeviceToDevice, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  b.release();
  b = bigger;
  bigger.p = nullptr;
  return GLOP_OK;
}

// Copies the n_alerts alerts (+ lines when wanted) and the counts to
// library-owned host arrays.
glop_status alerts_to_host(glop_ctx* c, const glop_alert* d_alerts, uint64_t n_alerts, const uint64_t* d_counts,
                           uint32_t k, uint64_t* counts, glop_alert** alerts, const uint64_t* d_lines, uint64_t** lines,
                           const uint64_t* d_lf, uint64_t* line_count) {
  glop_alert* a = static_cast<glop_alert*>(malloc(std::max<uint64_t>(n_alerts, 1) * sizeof(glop_alert)));
  uint64_t* l = lines ? static_cast<uint64_t*>(malloc(std::max<uint64_t>(n_alerts, 1) * 8)) : nullptr;
  cudaError_t e = a && (!lines || l) ? cudaSuccess : cudaErrorMemoryAllocation;
  if (e == cudaSuccess && n_alerts)
    e = cudaMemcpyAsync(a, d_alerts, n_alerts * sizeof(glop_alert), cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess && counts) e = cudaMemcpyAsync(counts, d_counts, (size_t)k * 8, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess && lines && n_alerts)
    e = cudaMemcpyAsync(l, d_lines, n_alerts * 8, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess && line_count) e = cudaMemcpyAsync(c->h_misc + 7, d_lf, 8, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    free(a);
    free(l);
    return fail(e == cudaErrorMemoryAllocation ? GLOP_ENOMEM : GLOP_ECUDA, cudaGetErrorString(e));
  }
  if (line_count) *line_count = c->h_misc[7] + 1;  // LineIndex::line_count() = 1 + LF bytes
  *alerts = a;
  if (lines) *lines = l;
  return GLOP_OK;
}

glop_status accum_begin(glop_ctx* c, Accum& A, uint32_t k, bool want_lines) {
  A.total = A.hits = 0;
  A.k = k;
  A.want_lines = want_lines;
  TRY(A.cnt.ensure((size_t)(2 * k + 3) * 8));
  CU(cudaMemsetAsync(A.cnt.p, 0, (size_t)(2 * k + 3) * 8, c->stream));
  TRY(A.alerts.ensure(std::max<size_t>(A.alerts.bytes, (1 << 16) * sizeof(glop_alert))));
  return GLOP_OK;
}

// One window: d_text = global [base, base + rd), starts [base, base + own).
glop_status accum_window(glop_ctx* c, const glop_trie* t, const glop_rules* r, Accum& A, const uint8_t* d_text,
                         uint64_t rd, uint64_t own, uint64_t base) {
  uint64_t nh = 0, kept = 0;
  for (;;) {
    const uint64_t room = A.alerts.bytes / sizeof(glop_alert) - A.total;
    glop_status s = pipeline_device_impl(c, t, r, d_text, rd, own, base, nullptr, 0,
                                         A.alerts.as<glop_alert>() + A.total, room, A.d_window_counts(), &nh, &kept);
    if (s == GLOP_ECAPACITY && kept > room) {  // grow, keeping the alerts so far; redo the window
      TRY(grow_keep(c, A.alerts, std::max<uint64_t>(2 * A.alerts.bytes, (A.total + kept + (1 << 16)) * sizeof(glop_alert)),
                    A.total * sizeof(glop_alert)));
      continue;
    }
    if (s != GLOP_OK) return s;
    break;
  }
  if (A.want_lines) {  // LineIndex over the owned bytes of this window, offset by the earlier windows' LFs
    TRY(grow_keep(c, A.lines, (A.total + kept) * 8 + 8, A.total * 8));
    TRY(line_numbers_impl(c, d_text, own, base, A.alerts.as<glop_alert>() + A.total, sizeof(glop_alert), kept,
                          A.lines.as<uint64_t>() + A.total, A.d_lf(), A.d_lf()));
  }
  ++c->launches;
  add_u64_kernel<<<(A.k + 255) / 256 + 1, 256, 0, c->stream>>>(
      reinterpret_cast<unsigned long long*>(A.d_counts()),
      reinterpret_cast<const unsigned long long*>(A.d_window_counts()), A.k);
  CU(cudaGetLastError());
  A.hits += nh;
  A.total += kept;
  return GLOP_OK;
}

glop_status accum_end(glop_ctx* c, Accum& A, glop_alert** alerts, uint64_t* n_alerts, uint64_t* counts,
                      uint64_t* stage1_hits, uint64_t** lines, uint64_t* line_count) {
  if (stage1_hits) *stage1_hits = A.hits;
  TRY(alerts_to_host(c, A.alerts.as<glop_alert>(), A.total, A.d_counts(), A.k, counts, alerts,
                     A.lines.as<uint64_t>(), lines, A.d_lf(), line_count));
  *n_alerts = A.total;
  return GLOP_OK;
}

glop_status run_pipeline_streamed(glop_ctx* c, const glop_trie* t, const glop_rules* r, const uint8_t* h_text,
                                  uint64_t n, uint64_t own, uint64_t base, glop_alert** alerts,
                                  uint64_t* n_alerts, uint64_t* counts, uint64_t* stage1_hits,
                                  uint64_t** lines = nullptr, uint64_t* line_count = nullptr) {
  const uint64_t halo = std::max<uint64_t>(std::max<uint64_t>(t->info.max_depth, r->max_len), 1) - 1;
  const uint64_t chunks = (own + kStreamChunk - 1) / kStreamChunk;
  for (int b = 0; b < 2; ++b) TRY(c->sbuf[b].ensure(kStreamChunk + halo + 64));
  Accum& A = c->acc;  // kept across calls (buffers grow rarely)
  TRY(accum_begin(c, A, r->view.n_patterns, lines || line_count));
  // Pageable text (a std::string, a file read into memory): the driver would
  // stage it through its own pinned buffers on one thread (~11 GB/s here);
  // instead a stager thread copies chunks into a ring of kPinRing pinned
  // buffers (host thread pool, non-temporal stores: hostcopy.cpp), running
  // ahead of the DMA by up to kPinRing chunks, so the copy engine never waits
  // for the host.
  constexpr uint64_t kPinRing = 3;
  cudaPointerAttributes pa{};
  const bool pageable = cudaPointerGetAttributes(&pa, h_text) != cudaSuccess || pa.type == cudaMemoryTypeUnregistered;
  cudaGetLastError();  // (older drivers report unregistered memory as an error)
  if (pageable) {
    for (uint64_t b = 0; b < kPinRing; ++b) CU(cudaEventSynchronize(c->ev_pin[b]));  // (a previous call's DMAs)
    const size_t need = kStreamChunk + halo + 64;  // (the halo depends on the trie and rules)
    if (c->pin_bytes < need) {
      for (void*& q : c->pin)
        if (q) cudaFreeHost(q), q = nullptr;
      c->pin_bytes = 0;
      for (void*& q : c->pin) CU(cudaMallocHost(&q, need));
      c->pin_bytes = need;
    }
  }
  auto span = [&](uint64_t i, uint64_t* lo, uint64_t* rd) {
    *lo = i * kStreamChunk;
    *rd = std::min<uint64_t>(std::min<uint64_t>(kStreamChunk, own - *lo) + halo, n - *lo);
  };
  // staged: chunks copied into the ring; issued: chunks whose DMA is enqueued
  // (pin[i % kPinRing] is reusable once ev_pin of chunk i's DMA has fired)
  struct Ring {
    std::mutex mu;
    std::condition_variable cv;
    uint64_t staged = 0, issued = 0;
    bool stop = false, failed = false;
    double copy_ms = 0, wait_ms = 0;  // GLOP_STAGE_TIMING
    std::thread th;
    ~Ring() {
      {
        std::lock_guard<std::mutex> lk(mu);
        stop = true;
      }
      cv.notify_all();
      if (th.joinable()) th.join();
    }
  } ring;
  if (pageable)
    ring.th = std::thread([&] {
      for (uint64_t i = 0; i < chunks; ++i) {
        const uint64_t b = i % kPinRing;
        if (i >= kPinRing) {  // wait for chunk i - kPinRing's DMA to be enqueued, then done
          std::unique_lock<std::mutex> lk(ring.mu);
          ring.cv.wait(lk, [&] { return ring.stop || ring.issued > i - kPinRing; });
          if (ring.stop) return;
          lk.unlock();
          if (cudaEventSynchronize(c->ev_pin[b]) != cudaSuccess) {
            std::lock_guard<std::mutex> lk2(ring.mu);
            ring.failed = true;
            ring.cv.notify_all();
            return;
          }
        }
        uint64_t lo, rd;
        span(i, &lo, &rd);
        const auto t0 = std::chrono::steady_clock::now();
        parallel_memcpy(c->pin[b], h_text + lo, rd);
        ring.copy_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        std::lock_guard<std::mutex> lk(ring.mu);
        ring.staged = i + 1;
        ring.cv.notify_all();
      }
    });
  auto dma = [&](uint64_t i) -> glop_status {
    uint64_t lo, rd;
    span(i, &lo, &rd);
    const void* src = h_text + lo;
    if (pageable) {
      const auto t0 = std::chrono::steady_clock::now();
      std::unique_lock<std::mutex> lk(ring.mu);
      ring.cv.wait(lk, [&] { return ring.staged > i || ring.failed; });
      ring.wait_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      if (ring.staged <= i) return fail(GLOP_ECUDA, "run_pfac_pipeline: staging copy failed");
      src = c->pin[i % kPinRing];
    }
    CU(cudaStreamWaitEvent(c->cstream, c->ev_free[i & 1], 0));
    CU(cudaMemcpyAsync(c->sbuf[i & 1].p, src, rd, cudaMemcpyHostToDevice, c->cstream));
    CU(cudaEventRecord(c->ev_copied[i & 1], c->cstream));
    if (pageable) {
      CU(cudaEventRecord(c->ev_pin[i % kPinRing], c->cstream));
      std::lock_guard<std::mutex> lk(ring.mu);
      ring.issued = i + 1;
      ring.cv.notify_all();
    }
    return GLOP_OK;
  };
  // ev_free[b]: device buffer b may be overwritten (recorded after its chunk's work)
  CU(cudaEventRecord(c->ev_free[0], c->stream));
  CU(cudaEventRecord(c->ev_free[1], c->stream));
  TRY(dma(0));
  for (uint64_t i = 0; i < chunks; ++i) {
    if (i + 1 < chunks) TRY(dma(i + 1));
    const uint64_t lo = i * kStreamChunk, own_i = std::min<uint64_t>(kStreamChunk, own - lo);
    const uint64_t rd = std::min<uint64_t>(own_i + halo, n - lo);
    CU(cudaStreamWaitEvent(c->stream, c->ev_copied[i & 1], 0));
    TRY(accum_window(c, t, r, A, c->sbuf[i & 1].as<uint8_t>(), rd, own_i, base + lo));
    CU(cudaEventRecord(c->ev_free[i & 1], c->stream));
  }
  if (pageable && getenv("GLOP_STAGE_TIMING"))
    fprintf(stderr, "staging: %llu chunks, copies %.1f ms, DMA issue waited %.1f ms\n", (unsigned long long)chunks,
            ring.copy_ms, ring.wait_ms);
  return accum_end(c, A, alerts, n_alerts, counts, stage1_hits, lines, line_count);
}

// Device LineIndex (lines.cuh): lines[i] = line of record i's offset (u64
// at byte 0 of each `stride`-byte record) in text d_text = global [base, base+n),
// plus *d_line_base when given (lines of earlier streamed chunks).  d_lf_acc
// (optional) is incremented by the number of LF bytes in text[0, n).
glop_status line_numbers_impl(glop_ctx* c, const uint8_t* d_text, uint64_t n, uint64_t base, const void* d_recs,
                              uint32_t stride, uint64_t count, uint64_t* d_lines,
                              const uint64_t* d_line_base, uint64_t* d_lf_acc) {
  if (count == 0 && !d_lf_acc) return GLOP_OK;
  if (n == 0) {
    if (count) {
      ++c->launches;
      lines_fill_kernel<<<1, 256, 0, c->stream>>>(reinterpret_cast<unsigned long long*>(d_lines), count,
                                                  reinterpret_cast<const unsigned long long*>(d_line_base));
      CU(cudaGetLastError());
    }
    return GLOP_OK;
  }
  const uint32_t a = (uint32_t)((uintptr_t)d_text & 15);
  const uint64_t nblocks = (n + a + kLineBlock - 1) / kLineBlock;
  TRY(c->lcount.ensure(nblocks * 8));
  TRY(c->lprefix.ensure(nblocks * 8));
  const uint8_t* A = d_text - a;
  const uint32_t grid = (uint32_t)std::min<uint64_t>((nblocks + 7) / 8, 16u * c->num_sms);
  c->launches += 2;
  lf_block_count_kernel<<<grid, 256, 0, c->stream>>>(A, a, n, nblocks, c->lcount.as<unsigned long long>());
  CU(cudaGetLastError());
  size_t tmp = 0;
  CU(cub::DeviceScan::ExclusiveSum(nullptr, tmp, c->lcount.as<unsigned long long>(),
                                   c->lprefix.as<unsigned long long>(), (int64_t)nblocks, c->stream));
  TRY(c->cub_tmp.ensure(tmp));
  CU(cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, tmp, c->lcount.as<unsigned long long>(),
                                   c->lprefix.as<unsigned long long>(), (int64_t)nblocks, c->stream));
  if (count) {
    ++c->launches;
    const uint32_t g2 = (uint32_t)std::min<uint64_t>((count + 7) / 8, 16u * c->num_sms);
    lines_of_kernel<<<g2, 256, 0, c->stream>>>(A, a, base, c->lprefix.as<unsigned long long>(), d_recs, stride, count,
                                               reinterpret_cast<unsigned long long*>(d_lines),
                                               reinterpret_cast<const unsigned long long*>(d_line_base));
    CU(cudaGetLastError());
  }
  if (d_lf_acc) {
    ++c->launches;
    lf_total_add_kernel<<<1, 1, 0, c->stream>>>(c->lcount.as<unsigned long long>(), c->lprefix.as<unsigned long long>(),
                                                nblocks, reinterpret_cast<unsigned long long*>(d_lf_acc));
    CU(cudaGetLastError());
  }
  return GLOP_OK;
}

// chunked_ac_scan's result (scan.hpp:207-243) from the exact occurrence
// list: chunk k = [k*c, (k+1)*c) is walked from the root over
// [k*c, min(k*c + c + overlap, n)), so it reports exactly the occurrences
// whose start it owns and whose end it reaches.
struct AcOwned {
  unsigned long long c, overlap, n;
  __host__ __device__ bool operator()(const DevHit& h) const {
    const unsigned long long own_begin = h.offset / c * c;
    const unsigned long long scan_end = own_begin + c + overlap < n ? own_begin + c + overlap : n;
    return h.offset + h.len <= scan_end;
  }
};

glop_status chunked_ac_impl(glop_ctx* c, const glop_trie* t, const uint8_t* d_text, uint64_t n, uint64_t chunk,
                            uint64_t overlap, glop_hit* d_out, uint64_t cap, uint64_t* n_out) {
  *n_out = 0;
  if (n == 0 || t->empty) return GLOP_OK;
  uint64_t hcap = std::max<uint64_t>(1 << 16, c->keys_alt.bytes / sizeof(glop_hit));
  TRY(c->keys_alt.ensure(hcap * sizeof(glop_hit)));
  uint64_t nh = 0;
  glop_status s = pfac_scan_device_impl(c, t, d_text, n, n, 0, GLOP_PFAC_AUTO, c->keys_alt.as<glop_hit>(), hcap, &nh);
  if (s == GLOP_ECAPACITY && nh > hcap) {
    c->keys_alt.release();
    hcap = nh;
    TRY(c->keys_alt.ensure(hcap * sizeof(glop_hit)));
    s = pfac_scan_device_impl(c, t, d_text, n, n, 0, GLOP_PFAC_AUTO, c->keys_alt.as<glop_hit>(), hcap, &nh);
  }
  if (s != GLOP_OK) return s;
  if (nh == 0) return GLOP_OK;
  if (nh > cap) {  // the selection is <= nh: size the output for the worst case
    *n_out = nh;
    return fail(GLOP_ECAPACITY, "chunked_ac_scan: output capacity");
  }
  const AcOwned pred{chunk ? chunk : std::max<uint64_t>(n, 1), overlap, n};
  TRY(c->misc.ensure(64));
  auto* d_sel = c->misc.as<unsigned long long>() + 7;
  const auto* in = reinterpret_cast<const DevHit*>(c->keys_alt.p);
  auto* out = reinterpret_cast<DevHit*>(d_out);
  size_t tmp = 0;
  CU(cub::DeviceSelect::If(nullptr, tmp, in, out, d_sel, (int64_t)nh, pred, c->stream));
  TRY(c->cub_tmp.ensure(tmp));
  CU(cub::DeviceSelect::If(c->cub_tmp.p, tmp, in, out, d_sel, (int64_t)nh, pred, c->stream));
  ++c->launches;
  TRY(sync_read(c, d_sel, 8));
  *n_out = c->h_misc[0];
  return GLOP_OK;
}

// The reference's kmp_search loop verbatim on one device thread (kmp.hpp:41-69)
// for inputs the chunk-parallel DFA cannot take: a failure table that is not
// the pattern's prefix function, or a pattern of 8,192 bytes or more.
__global__ void kmp_seq_kernel(const uint8_t* text, unsigned long long n, const uint8_t* p, uint32_t m,
                               const uint32_t* table, unsigned long long* out, unsigned long long cap,
                               unsigned long long* status) {
  unsigned long long found = 0, cmp = 0;
  uint32_t j = 0;
  for (unsigned long long i = 0; i < n; ++i) {
    const uint8_t b = text[i];
    for (;;) {
      ++cmp;
      if (b == p[j]) {
        ++j;
        if (j == m) {
          if (found < cap) out[found] = i + 1 - m;
          ++found;
          j = table[m - 1];
        }
        break;
      }
      if (j == 0) break;
      j = table[j - 1];
    }
  }
  status[0] = found;
  status[1] = cmp;
}

glop_status kmp_seq_impl(glop_ctx* c, const uint8_t* pat, uint32_t m, const uint32_t* fail_tab, const uint8_t* d_text,
                         uint64_t n, uint64_t* d_out, uint64_t cap, uint64_t* n_offsets, uint64_t* comparisons) {
  for (uint32_t i = 0; i < m; ++i)
    if (fail_tab[i] >= m) return fail(GLOP_EINVAL, "kmp_search: failure table entry out of range");
  TRY(c->kmp_dfa.ensure((size_t)m * 4 + m + 16));
  auto* d_tab = c->kmp_dfa.as<uint32_t>();
  auto* d_pat = reinterpret_cast<uint8_t*>(d_tab + m);
  CU(cudaMemcpyAsync(d_tab, fail_tab, (size_t)m * 4, cudaMemcpyHostToDevice, c->stream));
  CU(cudaMemcpyAsync(d_pat, pat, m, cudaMemcpyHostToDevice, c->stream));
  TRY(c->misc.ensure(64));
  ++c->launches;
  kmp_seq_kernel<<<1, 1, 0, c->stream>>>(d_text, n, d_pat, m, d_tab, reinterpret_cast<unsigned long long*>(d_out),
                                         cap, c->misc.as<unsigned long long>());
  CU(cudaGetLastError());
  TRY(sync_read(c, c->misc.p, 16));
  *n_offsets = c->h_misc[0];
  if (comparisons) *comparisons += c->h_misc[1];
  if (*n_offsets > cap) return fail(GLOP_ECAPACITY, "kmp_search: output capacity");
  return GLOP_OK;
}

glop_status pipeline_host(glop_ctx* c, const glop_trie* t, const glop_rules* r, const uint8_t* text, uint64_t n,
                          uint64_t own, uint64_t base, int text_on_device, glop_alert** alerts, uint64_t* n_alerts,
                          uint64_t* counts, uint64_t* stage1_hits, uint64_t** lines, uint64_t* line_count);

}  // namespace

// ============================================================== C ABI
extern "C" {

const char* glop_last_error(void) { return g_err.c_str(); }
const char* glop_version(void) { return "glop-b200 0.1 (sm_100a)"; }

glop_status glop_ctx_create(int device, glop_ctx** out) {
  *out = nullptr;
  int count = 0;
  CU(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count) return fail(GLOP_EINVAL, "glop_ctx_create: bad device");
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    return fail(GLOP_ECUDA, std::string("glop: needs an sm_100 device, found ") + prop.name);
  Dev g(device);
  auto* c = new glop_ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  c->smem_optin = prop.sharedMemPerBlockOptin;
  cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMallocHost(&c->h_misc, 64);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev1);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&c->ev_copied[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_free[i], cudaEventDisableTiming);
  }
  for (int i = 0; i < 3 && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&c->ev_pin[i], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) {
    delete c;
    return fail(GLOP_ECUDA, cudaGetErrorString(e));
  }
  *out = c;
  return GLOP_OK;
}

glop_status glop_ctx_destroy(glop_ctx* c) {
  if (!c) return GLOP_OK;
  Dev g(c->device);
  cudaStreamSynchronize(c->stream);
  for (DBuf* b : {&c->text, &c->staging, &c->out, &c->dir, &c->prefix, &c->misc, &c->keys,
                  &c->keys_alt, &c->cub_tmp, &c->keep, &c->bcounts, &c->bprefix, &c->alerts,
                  &c->kmp_dfa, &c->spill, &c->sbuf[0], &c->sbuf[1], &c->lcount, &c->lprefix, &c->loffs,
                  &c->kcounts, &c->keep8, &c->counts_tmp, &c->palerts, &c->plines})
    b->release();
  c->acc.release();
  if (c->cstream) {
    cudaStreamSynchronize(c->cstream);
    cudaStreamDestroy(c->cstream);
  }
  for (int i = 0; i < 2; ++i) {
    if (c->ev_copied[i]) cudaEventDestroy(c->ev_copied[i]);
    if (c->ev_free[i]) cudaEventDestroy(c->ev_free[i]);
  }
  for (cudaEvent_t e : c->ev_pin)
    if (e) cudaEventDestroy(e);
  cudaFreeHost(c->h_misc);
  for (void* p : c->pin)
    if (p) cudaFreeHost(p);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  cudaStreamDestroy(c->stream);
  delete c;
  return GLOP_OK;
}

void* glop_ctx_stream(glop_ctx* c) { return c ? (void*)c->stream : nullptr; }

glop_status glop_ctx_synchronize(glop_ctx* c) {
  Dev g(c->device);
  CU(cudaStreamSynchronize(c->stream));
  return GLOP_OK;
}

glop_status glop_trie_upload(glop_ctx* c, const int32_t* dense, uint32_t Q, const uint32_t* out_off,
                             const glop_output* out_flat, glop_trie** out) {
  *out = nullptr;
  if (!c || !dense || !out_off || Q == 0) return fail(GLOP_EINVAL, "glop_trie_upload: null/empty input");
  if (Q >= 0x7FFFFFFFu) return fail(GLOP_EINVAL, "glop_trie_upload: too many states");
  // --- structure: BFS from the root, every non-root state exactly one parent
  std::vector<uint32_t> depth(Q, 0);
  std::vector<uint8_t> seen(Q, 0);
  std::vector<uint32_t> order;
  order.reserve(Q);
  order.push_back(0);
  seen[0] = 1;
  bool used[256] = {};
  for (size_t h = 0; h < order.size(); ++h) {
    const uint32_t s = order[h];
    for (int b = 0; b < 256; ++b) {
      const int32_t t = dense[(size_t)s * 256 + b];
      if (t == -1) continue;
      if (t <= 0 || (uint32_t)t >= Q || seen[t])
        return fail(GLOP_EINVAL, "glop_trie_upload: not a failureless trie");
      seen[t] = 1;
      depth[t] = depth[s] + 1;
      used[b] = true;
      order.push_back((uint32_t)t);
    }
  }
  if (order.size() != Q) return fail(GLOP_EINVAL, "glop_trie_upload: unreachable state");
  const uint32_t n_out = out_off[Q];
  if (n_out && !out_flat) return fail(GLOP_EINVAL, "glop_trie_upload: null outputs");
  uint32_t lmin = 0, lmax = 0, max_pid = 0;
  std::vector<uint8_t> has_out(Q, 0);
  for (uint32_t s = 0; s < Q; ++s) {
    if (out_off[s + 1] < out_off[s]) return fail(GLOP_EINVAL, "glop_trie_upload: bad out_offsets");
    if (s == 0) continue;  // the walk never emits at the root (scan.hpp:126)
    if (out_off[s + 1] > out_off[s]) {
      has_out[s] = 1;
      lmin = lmin ? std::min(lmin, depth[s]) : depth[s];
      lmax = std::max(lmax, depth[s]);
    }
  }
  // compact out lists: drop root outputs, keep the CSR for states 1..Q-1
  std::vector<uint32_t> off2(Q + 1, 0), pid2;
  for (uint32_t s = 0; s < Q; ++s) {
    off2[s] = (uint32_t)pid2.size();
    if (s == 0) continue;
    for (uint32_t o = out_off[s]; o < out_off[s + 1]; ++o) {
      pid2.push_back(out_flat[o].pattern_id);
      max_pid = std::max(max_pid, out_flat[o].pattern_id);
    }
  }
  off2[Q] = (uint32_t)pid2.size();
  std::vector<uint32_t> pid_len(pid2.empty() ? 1 : (size_t)max_pid + 1, 0xFFFFFFFFu);
  for (uint32_t s = 1; s < Q; ++s)
    for (uint32_t o = out_off[s]; o < out_off[s + 1]; ++o) {
      uint32_t& L = pid_len[out_flat[o].pattern_id];
      if (L != 0xFFFFFFFFu && L != out_flat[o].matched_len)
        return fail(GLOP_EINVAL, "glop_trie_upload: pattern id with two lengths");
      L = out_flat[o].matched_len;
    }
  // most hits one start position emits: outputs summed along a root path
  // (BFS order visits parents first); a pfac8 lane checks up to 4 starts
  uint32_t max_emits = 0;
  {
    std::vector<uint32_t> cum(Q, 0);
    for (size_t h = 0; h < order.size(); ++h) {
      const uint32_t s = order[h];
      max_emits = std::max(max_emits, cum[s]);
      for (int b = 0; b < 256; ++b) {
        const int32_t t2 = dense[(size_t)s * 256 + b];
        if (t2 > 0) cum[t2] = cum[s] + (off2[t2 + 1] - off2[t2]);
      }
    }
  }
  // --- alphabet classes (ascending byte order; class 0 = no edge anywhere)
  // (all 256 bytes on edges: the identity map, 256 classes -- no byte needs
  // the "no edge" class, and 257 classes would not fit the u8 map)
  uint8_t cls[256];
  uint32_t C = 1;
  for (int b = 0; b < 256; ++b) C += used[b];
  if (C == 257) {
    C = 256;
    for (int b = 0; b < 256; ++b) cls[b] = (uint8_t)b;
  } else {
    C = 1;
    for (int b = 0; b < 256; ++b) cls[b] = used[b] ? (uint8_t)C++ : 0;
  }
  const bool u16 = Q < 0x8000u;
  const size_t eb = u16 ? 2 : 4;
  const size_t table_bytes = up16((size_t)Q * C * eb);
  std::vector<uint8_t> table(table_bytes, 0);
  for (uint32_t s = 0; s < Q; ++s)
    for (int b = 0; b < 256; ++b) {
      const int32_t t = dense[(size_t)s * 256 + b];
      if (t < 0) continue;
      const size_t idx = (size_t)s * C + cls[b];
      if (u16) {
        uint16_t e = (uint16_t)(t | (has_out[t] ? 0x8000u : 0));
        memcpy(&table[idx * 2], &e, 2);
      } else {
        uint32_t e = (uint32_t)t | (has_out[t] ? 0x80000000u : 0);
        memcpy(&table[idx * 4], &e, 4);
      }
    }
  // --- filter tables: root paths of length lmin (q-gram d-mask) and of
  // length J = min(lmin, 8) (jump table + level-2 bitmap)
  const uint32_t q = lmin ? std::min<uint32_t>(4, lmin) : 1;
  const uint32_t stride = lmin ? std::min<uint32_t>(lmin - q + 1, 8) : 1;
  const uint32_t J = lmin ? std::min<uint32_t>(lmin, 8) : 1;
  std::vector<uint8_t> dmask(kDmaskBytes, 0);
  std::vector<uint32_t> bm2(kBm2Bits / 32, 0), bm28((1u << kP8Bm2Log2) / 32, 0);
  // pfac8 level 1 (outputs only at depth >= 8): bit d-1 of the bucket of the
  // 4-gram at offset d (1..4) of every 8-byte root path
  std::vector<uint8_t> dmask8(kP8DmaskBytes, 0);
  std::vector<unsigned long long> grams8;  // ((prev top byte, cur) << 2 | d-1) of every 8-byte root path
  const bool p8 = lmin >= 8;
  bool bits8 = false, bloom2 = false, two8 = false, lane8 = false, lists8 = false;
  // visits every root path of length `depth`: cb(path bytes, end state)
  auto for_paths = [&](uint32_t depth, auto&& cb) {
    std::vector<uint8_t> path(depth + 1);
    std::vector<uint32_t> st(depth + 1, 0);
    std::vector<int> nb(depth + 1, 0);
    int d = 0;
    while (d >= 0) {
      if ((uint32_t)d == depth) {
        cb(path.data(), st[d]);
        --d;
        continue;
      }
      bool pushed = false;
      while (nb[d] < 256) {
        const int b = nb[d]++;
        const int32_t tt = dense[(size_t)st[d] * 256 + b];
        if (tt < 0) continue;
        path[d] = (uint8_t)b;
        st[d + 1] = (uint32_t)tt;
        nb[d + 1] = 0;
        ++d;
        pushed = true;
        break;
      }
      if (!pushed) --d;
    }
  };
  std::vector<JumpEntry> jump;
  uint32_t cap_log2 = 6;
  if (lmin) {
    for_paths(lmin, [&](const uint8_t* path, uint32_t) {
      for (uint32_t k = 0; k < stride; ++k) {
        uint32_t g = 0;
        for (uint32_t x = 0; x < q; ++x) g |= (uint32_t)path[k + x] << (8 * x);
        dmask[qgram_bucket(g, q)] |= (uint8_t)(1u << k);
      }
    });
    std::vector<std::pair<unsigned long long, uint32_t>> keys;
    for_paths(J, [&](const uint8_t* path, uint32_t s) {
      unsigned long long key = 0;
      for (uint32_t x = 0; x < J; ++x) key |= (unsigned long long)path[x] << (8 * x);
      keys.push_back({key, s});
      if (p8)
        for (uint32_t d = 1; d <= 4; ++d) {
          // (prev's top byte, cur) of the gram at offset d: 40 bits, << 2 | d - 1
          const uint32_t prev_top = (uint32_t)(key >> (8 * (d - 1))) & 0xFFu, cur = (uint32_t)(key >> (8 * d));
          grams8.push_back(((unsigned long long)prev_top << 32 | cur) << 2 | (d - 1));
        }
      const uint32_t bit = prefix_bit(key);
      bm2[bit >> 5] |= 1u << (bit & 31);
      const uint32_t bit8 = prefix_hash32((uint32_t)key, (uint32_t)(key >> 32)) >> (32 - kP8Bm2Log2);
      bm28[bit8 >> 5] |= 1u << (bit8 & 31);
    });
    if (p8) {
      std::sort(grams8.begin(), grams8.end());
      grams8.erase(std::unique(grams8.begin(), grams8.end()), grams8.end());
      const char* env = getenv("GLOP_P8_BITS_MIN");  // experiments: override the layout threshold
      bits8 = grams8.size() > (env ? (size_t)atoll(env) : (size_t)kP8BitsGrams);
      const char* env3 = getenv("GLOP_P8_LANE_MAX");  // experiments: override the lane-replicated threshold
      const char* env4 = getenv("GLOP_P8_LANE_MIN");
      lane8 = grams8.size() <= (env3 ? (size_t)atoll(env3) : (size_t)kP8LaneGrams) &&
              grams8.size() > (env4 ? (size_t)atoll(env4) : (size_t)kP8LaneMinGrams);
      const char* env2 = getenv("GLOP_P8_BITS2_MIN");  // experiments: override the two-bit threshold
      two8 = bits8 && grams8.size() > (env2 ? (size_t)atoll(env2) : (size_t)kP8Bits2Grams);
      for (unsigned long long x : grams8) {
        const uint32_t cur = (uint32_t)(x >> 2), prev = (uint32_t)(x >> 34) << 24, bit = 1u << (x & 3);
        if (lane8) {  // the gram's bit in every lane's copy of its word
          const uint32_t w = p8_lane_off(prev, cur), b1 = p8_bit1(cur) & 31u;
          for (uint32_t l = 0; l < 32; ++l) dmask8[w + 4 * l + (b1 >> 3)] |= (uint8_t)(1u << (b1 & 7));
        } else if (bits8) {  // little-endian bits of the u32 words
          const bool pv = two8 && GLOP_P8_BIT2_PRMT;  // (must match p8_dmask)
          const uint32_t w = pv ? p8_word_off2(prev, cur) : p8_word_off(prev, cur);
          const uint32_t b1 = p8_bit1(cur) & 31u;
          dmask8[w + (b1 >> 3)] |= (uint8_t)(1u << (b1 & 7));
          if (two8) {  // second bit in the same 32-bit word
            const uint32_t b2 = (pv ? p8_pb2(prev, cur) : p8_bit2(cur)) & 31u;
            dmask8[w + (b2 >> 3)] |= (uint8_t)(1u << (b2 & 7));
          }
        } else {
          dmask8[p8_byte_off(prev, cur)] |= (uint8_t)bit;
        }
      }
    }
    if (p8) {  // large prefix sets: a second level-2 bit per prefix
      const char* env = getenv("GLOP_P8_BLOOM2_MIN");  // experiments: override the threshold
      bloom2 = bits8 && !lane8 && keys.size() > (env ? (size_t)atoll(env) : (size_t)kP8Bloom2Keys);
      if (bloom2)
        for (const auto& kv : keys) {
          const uint32_t bit = prefix_bit2(kv.first);
          bm2[bit >> 5] |= 1u << (bit & 31);
          const uint32_t bit8 =
              prefix_hash2(prefix_hash32((uint32_t)kv.first, (uint32_t)(kv.first >> 32))) >> (32 - kP8Bm2Log2);
          bm28[bit8 >> 5] |= 1u << (bit8 & 31);
        }
    }
    // A sparse table: every probe past the first is a dependent L2 round
    // trip, and a false survivor's probes run to an empty slot.  Load factor
    // <= 1/16 up to 4,096 prefixes, 1/8 up to 65,536, then 1/4 (measured
    // against 1/2: k=1,000 2.241 -> 2.191 ms, k=10,000 2.699 -> 2.665 ms, DPI
    // 1.618 -> 1.620 ms; the table stays L2-resident: 1 MB at 4,096 prefixes)
    const char* env_lf = getenv("GLOP_JUMP_SPARSE");  // experiments: fixed factor
    // (pfac8 automata only: the general kernel keeps 1/2, so its table still
    // fits in shared memory where it did)
    const size_t sparse = env_lf ? (size_t)atoll(env_lf)
                          : !p8 ? 2 : keys.size() <= 4096 ? 16 : keys.size() <= 65536 ? 8 : 4;
    while ((1ull << cap_log2) < sparse * keys.size()) ++cap_log2;
    jump.assign(1ull << cap_log2, JumpEntry{0, 0, 0});
    const uint32_t mask = (1u << cap_log2) - 1;
    for (const auto& [key, s] : keys) {
      uint32_t h = jump_slot(key, cap_log2);
      while (jump[h].state1) h = (h + 1) & mask;
      const uint32_t no = off2[s + 1] - off2[s];
      jump[h] = JumpEntry{key, s + 1, jump_out(pid2.data(), off2[s], no)};
      lists8 = lists8 || (jump[h].out >= kOutList && jump[h].out != kOutNone && jump[h].out != kOutMany);
    }
  } else {
    jump.assign(1ull << cap_log2, JumpEntry{0, 0, 0});
  }
  const size_t jump_bytes = jump.size() * sizeof(JumpEntry);
  // --- one device allocation
  const size_t o_cls = 0, o_table = 256, o_off = o_table + table_bytes;
  const size_t o_pid = o_off + up16((size_t)(Q + 1) * 4);
  const size_t o_plen = o_pid + up16(std::max<size_t>(pid2.size(), 1) * 4);
  const size_t o_dmask = o_plen + up16(pid_len.size() * 4);
  const size_t o_bm2 = o_dmask + kDmaskBytes;
  const size_t o_bm28 = o_bm2 + kBm2Bytes;
  const size_t o_dmask8 = o_bm28 + kP8Bm2Bytes;
  const size_t o_jump = o_dmask8 + kP8DmaskBytes;
  const size_t total = o_jump + jump_bytes;
  std::vector<uint8_t> host(total, 0);
  memcpy(&host[o_cls], cls, 256);
  memcpy(&host[o_table], table.data(), table_bytes);
  memcpy(&host[o_off], off2.data(), (Q + 1) * 4);
  if (!pid2.empty()) memcpy(&host[o_pid], pid2.data(), pid2.size() * 4);
  memcpy(&host[o_plen], pid_len.data(), pid_len.size() * 4);
  memcpy(&host[o_dmask], dmask.data(), kDmaskBytes);
  memcpy(&host[o_bm2], bm2.data(), kBm2Bytes);
  memcpy(&host[o_bm28], bm28.data(), kP8Bm2Bytes);
  memcpy(&host[o_dmask8], dmask8.data(), kP8DmaskBytes);
  memcpy(&host[o_jump], jump.data(), jump_bytes);
  Dev g(c->device);
  void* mem = nullptr;
  CU(cudaMalloc(&mem, total));
  cudaError_t e = cudaMemcpy(mem, host.data(), total, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(mem);
    return fail(GLOP_ECUDA, cudaGetErrorString(e));
  }
  auto* t = new glop_trie();
  t->device = c->device;
  t->mem = mem;
  uint8_t* m = static_cast<uint8_t*>(mem);
  t->view.cls = m + o_cls;
  t->view.table = m + o_table;
  t->view.out_off = reinterpret_cast<const uint32_t*>(m + o_off);
  t->view.out_pid = reinterpret_cast<const uint32_t*>(m + o_pid);
  t->view.pid_len = reinterpret_cast<const uint32_t*>(m + o_plen);
  t->view.dmask = m + o_dmask;
  t->view.bm2 = reinterpret_cast<const uint32_t*>(m + o_bm2);
  t->view.bm2_8 = reinterpret_cast<const uint32_t*>(m + o_bm28);
  t->view.jump = reinterpret_cast<const JumpEntry*>(m + o_jump);
  t->view.dmask8 = m + o_dmask8;
  t->p8 = p8;
  t->p8_l1 = lane8 ? 4 : two8 && bloom2 ? (lists8 ? 5 : 3) : bloom2 ? 2 : bits8 ? 1 : 0;
  t->p8_lane_emits = 4 * max_emits;
  t->p8_careful = t->p8_lane_emits > kP8Hits - GLOP_P8_FLUSH_AT || getenv("GLOP_P8_CAREFUL");
  t->view.jump_depth = J;
  t->view.jump_cap_log2 = cap_log2;
  t->view.jump_bytes = (uint32_t)jump_bytes;
  t->view.Q = Q;
  t->view.C = C;
  t->view.lmin = lmin;
  t->view.lmax = lmax;
  t->view.q = q;
  t->view.stride = stride;
  t->view.table_bytes = (uint32_t)std::min<size_t>(table_bytes, 0xFFFFFFFFu);
  t->empty = pid2.empty();
  t->u16 = u16;
  t->max_pid = max_pid;
  const size_t cap = std::min<size_t>(kSmemMax, c->smem_optin ? c->smem_optin : kSmemMax);
  // shared-memory placement, most valuable first: jump table, then the
  // transition table (filtered kernel); transition table (direct kernel)
  t->smem_jump = make_warp_layout(true, (uint32_t)jump_bytes, 0).total <= cap;
  t->smem_filter = make_warp_layout(true, t->smem_jump ? (uint32_t)jump_bytes : 0, (uint32_t)table_bytes).total <= cap;
  t->smem_direct = make_warp_layout(false, 0, (uint32_t)table_bytes).total <= cap;
  t->info = glop_trie_info{Q, C, lmin, lmax, q, stride, (uint32_t)eb, t->smem_filter ? 1u : 0u,
                           (uint64_t)table_bytes, J, t->smem_jump ? 1u : 0u, (uint32_t)jump.size(), 0u};
  *out = t;
  return GLOP_OK;
}

glop_status glop_trie_destroy(glop_trie* t) {
  if (!t) return GLOP_OK;
  Dev g(t->device);
  cudaFree(t->mem);
  delete t;
  return GLOP_OK;
}

glop_status glop_trie_get_info(const glop_trie* t, glop_trie_info* info) {
  if (!t || !info) return fail(GLOP_EINVAL, "null");
  *info = t->info;
  return GLOP_OK;
}

glop_status glop_pfac_scan_device(glop_ctx* c, const glop_trie* t, const uint8_t* d_text, uint64_t n,
                                  uint64_t own, uint64_t base, glop_pfac_kernel kernel, glop_hit* d_out,
                                  uint64_t cap, uint64_t* n_hits) {
  if (!c || !t || !n_hits) return fail(GLOP_EINVAL, "glop_pfac_scan_device: null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  Dev g(c->device);
  return pfac_scan_device_impl(c, t, d_text, n, own, base, kernel, d_out, cap, n_hits);
}

glop_status glop_pfac_scan(glop_ctx* c, const glop_trie* t, const uint8_t* text, uint64_t n,
                           int text_on_device, glop_hit** hits, uint64_t* n_hits) {
  return glop_pfac_scan_shard(c, t, text, n, n, 0, text_on_device, hits, n_hits);
}

glop_status glop_pfac_scan_shard(glop_ctx* c, const glop_trie* t, const uint8_t* text, uint64_t n, uint64_t own,
                                 uint64_t base, int text_on_device, glop_hit** hits, uint64_t* n_hits) {
  if (!c || !t || !hits || !n_hits) return fail(GLOP_EINVAL, "glop_pfac_scan: null argument");
  if (own > n) return fail(GLOP_EINVAL, "glop_pfac_scan: own > n");
  std::lock_guard<std::mutex> lk(c->mu);
  Dev g(c->device);
  *hits = nullptr;
  *n_hits = 0;
  const uint8_t* d_text = nullptr;
  TRY(to_device_text(c, text, n, text_on_device, &d_text));
  uint64_t cap = std::max<uint64_t>(1 << 16, c->out.bytes / sizeof(glop_hit));
  TRY(c->out.ensure(cap * sizeof(glop_hit)));
  uint64_t total = 0;
  glop_status s = pfac_scan_device_impl(c, t, d_text, n, own, base, GLOP_PFAC_AUTO, c->out.as<glop_hit>(), cap, &total);
  if (s == GLOP_ECAPACITY && total > cap) {
    c->out.release();
    cap = total;
    TRY(c->out.ensure(cap * sizeof(glop_hit)));
    s = pfac_scan_device_impl(c, t, d_text, n, own, base, GLOP_PFAC_AUTO, c->out.as<glop_hit>(), cap, &total);
  }
  if (s != GLOP_OK) return s;
  glop_hit* h = static_cast<glop_hit*>(malloc(std::max<uint64_t>(total, 1) * sizeof(glop_hit)));
  if (!h) return fail(GLOP_ENOMEM, "glop_pfac_scan: host allocation");
  if (total) {
    cudaError_t e = cudaMemcpyAsync(h, c->out.p, total * sizeof(glop_hit), cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
      free(h);
      return fail(GLOP_ECUDA, cudaGetErrorString(e));
    }
  } else {
    CU(cudaStreamSynchronize(c->stream));
  }
  *hits = h;
  *n_hits = total;
  return GLOP_OK;
}

glop_status glop_rules_upload(glop_ctx* c, const uint8_t* bytes, const uint64_t* off, uint32_t k,
                              uint64_t prefix_len, glop_rules** out) {
  *out = nullptr;
  if (!c || !off) return fail(GLOP_EINVAL, "glop_rules_upload: null argument");
  if (prefix_len < 1) return fail(GLOP_EINVAL, "truncate_prefixes: prefix_len must be >= 1");
  const uint64_t nb = off[k];
  for (uint32_t i = 0; i < k; ++i)
    if (off[i + 1] < off[i]) return fail(GLOP_EINVAL, "glop_rules_upload: bad offsets");
  Dev g(c->device);
  const size_t o_off = up16(std::max<uint64_t>(nb, 1));
  const size_t total = o_off + (size_t)(k + 1) * 8;
  std::vector<uint8_t> host(total, 0);
  if (nb) memcpy(host.data(), bytes, nb);
  memcpy(&host[o_off], off, (size_t)(k + 1) * 8);
  void* mem = nullptr;
  CU(cudaMalloc(&mem, total));
  cudaError_t e = cudaMemcpy(mem, host.data(), total, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(mem);
    return fail(GLOP_ECUDA, cudaGetErrorString(e));
  }
  auto* r = new glop_rules();
  r->device = c->device;
  r->mem = mem;
  r->view.bytes = static_cast<uint8_t*>(mem);
  r->view.off = reinterpret_cast<const unsigned long long*>(static_cast<uint8_t*>(mem) + o_off);
  r->view.n_patterns = k;
  r->view.prefix_len = prefix_len;
  for (uint32_t i = 0; i < k; ++i) r->max_len = std::max<uint64_t>(r->max_len, off[i + 1] - off[i]);
  *out = r;
  return GLOP_OK;
}

glop_status glop_rules_destroy(glop_rules* r) {
  if (!r) return GLOP_OK;
  Dev g(r->device);
  cudaFree(r->mem);
  delete r;
  return GLOP_OK;
}

glop_status glop_verify_hits_device(glop_ctx* c, const glop_rules* r, const uint8_t* d_text, uint64_t n,
                                    uint64_t base, const glop_hit* d_hits, uint64_t n_hits, glop_alert* d_out,
                                    uint64_t* n_alerts, uint64_t* d_counts) {
  if (!c || !r || !n_alerts) return fail(GLOP_EINVAL, "glop_verify_hits_device: null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  Dev g(c->device);
  return verify_device_impl(c, r, d_text, n, base, d_hits, n_hits, d_out, n_alerts, d_counts);
}

glop_status glop_verify_hits(glop_ctx* c, const glop_rules* r, const uint8_t* text, uint64_t n,
                             int text_on_device, const glop_hit* hits, uint64_t n_hits, int hits_on_device,
                             glop_alert** alerts, uint64_t* n_alerts, uint64_t* counts) {
  if (!c || !r || !alerts || !n_alerts) return fail(GLOP_EINVAL, "glop_verify_hits: null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  Dev g(c->device);
  *alerts = nullptr;
  *n_alerts = 0;
  const uint8_t* d_text = nullptr;
  TRY(to_device_text(c, text, n, text_on_device, &d_text));
  const glop_hit* d_hits = hits;
  if (!hits_on_device && n_hits) {
    TRY(c->out.ensure(n_hits * sizeof(glop_hit)));
    CU(cudaMemcpyAsync(c->out.p, hits, n_hits * sizeof(glop_hit), cudaMemcpyHostToDevice, c->stream));
    d_hits = c->out.as<glop_hit>();
  }
  TRY(c->alerts.ensure(std::max<uint64_t>(n_hits, 1) * sizeof(glop_alert) + (size_t)(r->view.n_patterns + 1) * 8));
  glop_alert* d_alerts = c->alerts.as<glop_alert>();
  uint64_t* d_counts = nullptr;
  if (counts) {
    d_counts = reinterpret_cast<uint64_t*>(d_alerts + std::max<uint64_t>(n_hits, 1));
    CU(cudaMemsetAsync(d_counts, 0, (size_t)r->view.n_patterns * 8, c->stream));
  }
  uint64_t kept = 0;
  TRY(verify_device_impl(c, r, d_text, n, 0, d_hits, n_hits, d_alerts, &kept, d_counts));
  glop_alert* a = static_cast<glop_alert*>(malloc(std::max<uint64_t>(kept, 1) * sizeof(glop_alert)));
  if (!a) return fail(GLOP_ENOMEM, "glop_verify_hits: host allocation");
  cudaError_t e = cudaSuccess;
  if (kept) e = cudaMemcpyAsync(a, d_alerts, kept * sizeof(glop_alert), cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess && counts)
    e = cudaMemcpyAsync(counts, d_counts, (size_t)r->view.n_patterns * 8, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    free(a);
    return fail(GLOP_ECUDA, cudaGetErrorString(e));
  }
  *alerts = a;
  *n_alerts = kept;
  return GLOP_OK;
}

glop_status glop_kmp_search_device(glop_ctx* c, const uint8_t* p, uint32_t m, const uint32_t* failure,
                                   const uint8_t* d_text, uint64_t n, uint64_t own, uint64_t base,
                                   uint64_t* d_out, uint64_t cap, uint64_t* n_offsets,
                                   uint64_t* comparisons) {
  if (!c || !n_offsets || (m && (!p || !failure))) return fail(GLOP_EINVAL, "glop_kmp_search_device: null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  Dev g(c->device);
  return kmp_device_impl(c, p, m, failure, d_text, n, own, base, d_out, cap, n_offsets, comparisons);
}

glop_status glop_kmp_search_device_async(glop_ctx* c, const uint8_t* p, uint32_t m, const uint32_t* failure,
                                         const uint8_t* d_text, uint64_t n, uint64_t own, uint64_t base,
                                         uint64_t* d_out, uint64_t cap, glop_pipeline_ticket* ticket) {
  if (!c || !ticket || (m && (!p || !failure))) return fail(GLOP_EINVAL, "glop_kmp_search_device_async: null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  Dev g(c->device);
  memset(ticket, 0, sizeof *ticket);
  uint64_t no = 0, cmp = 0;
  const glop_status s = kmp_device_impl(c, p, m, failure, d_text, n, own, base, d_out, cap, &no, &cmp, 0, ticket);
  if (s != GLOP_OK || ticket->region == 0) {  // failed, or ran synchronously (empty, sequential walk)
    ticket->done = s == GLOP_OK ? 1 : 2;
    ticket->raw[0] = no;
    ticket->raw[2] = cmp;
    ticket->raw[7] = (uint64_t)s;
    ticket->stage2 = 3;
  }
  return s;
}

glop_status glop_kmp_ticket_result(const glop_pipeline_ticket* k, uint64_t* n_offsets, uint64_t* comparisons) {
  if (!k || !n_offsets) return fail(GLOP_EINVAL, "glop_kmp_ticket_result: null argument");
  if (k->done == 2) return fail((glop_status)k->raw[7], "kmp_search: failed");
  if (k->done == 0 && ((k->raw[1] & 1u) || k->raw[3] > k->region))
    return fail(GLOP_EAGAIN, "kmp_search: this input needs the synchronous path (match-dense tile / staging overflow)");
  *n_offsets = k->raw[0];
  if (comparisons) *comparisons += k->raw[2];
  if (*n_offsets > k->hit_cap && k->done == 0) return fail(GLOP_ECAPACITY, "kmp_search: output capacity");
  return GLOP_OK;
}

glop_status glop_kmp_search(glop_ctx* c, const uint8_t* p, uint32_t m, const uint32_t* failure,
                            const uint8_t* text, uint64_t n, int text_on_device, uint64_t** offsets,
                            uint64_t* n_offsets, uint64_t* comparisons) {
  return glop_kmp_search_shard(c, p, m, failure, text, n, 0, n, 0, text_on_device, offsets, n_offsets, comparisons);
}

glop_status glop_kmp_search_shard(glop_ctx* c, const uint8_t* p, uint32_t m, const uint32_t* failure,
                                  const uint8_t* text, uint64_t n, uint64_t skip, uint64_t own, uint64_t base,
                                  int text_on_device, uint64_t** offsets, uint64_t* n_offsets,
                                  uint64_t* comparisons) {
  if (!c || !offsets || !n_offsets || (m && (!p || !failure)))
    return fail(GLOP_EINVAL, "glop_kmp_search: null argument");
  if (own > n) return fail(GLOP_EINVAL, "glop_kmp_search: own > n");
  std::lock_guard<std::mutex> lk(c->mu);
  Dev g(c->device);
  *offsets = nullptr;
  *n_offsets = 0;
  const uint8_t* d_text = nullptr;
  if (m && n >= m) TRY(to_device_text(c, text, n, text_on_device, &d_text));
  uint64_t cap = std::max<uint64_t>(1 << 16, c->out.bytes / 8);
  TRY(c->out.ensure(cap * 8));
  uint64_t total = 0, cmp0 = comparisons ? *comparisons : 0;
  glop_status s =
      kmp_device_impl(c, p, m, failure, d_text, n, own, base, c->out.as<uint64_t>(), cap, &total, comparisons, skip);
  if (s == GLOP_ECAPACITY && total > cap) {
    c->out.release();
    cap = total;
    TRY(c->out.ensure(cap * 8));
    if (comparisons) *comparisons = cmp0;
    s = kmp_device_impl(c, p, m, failure, d_text, n, own, base, c->out.as<uint64_t>(), cap, &total, comparisons, skip);
  }
  if (s != GLOP_OK) return s;
  uint64_t* o = static_cast<uint64_t*>(malloc(std::max<uint64_t>(total, 1) * 8));
  if (!o) return fail(GLOP_ENOMEM, "glop_kmp_search: host allocation");
  cudaError_t e = cudaSuccess;
  if (total) e = cudaMemcpyAsync(o, c->out.p, total * 8, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    free(o);
    return fail(GLOP_ECUDA, cudaGetErrorString(e));
  }
  *offsets = o;
  *n_offsets = total;
  return GLOP_OK;
}

glop_status glop_build_failureless_trie(const uint8_t* bytes, const uint64_t* off, uint32_t k,
                                        uint64_t prefix_len, uint64_t max_states, int32_t** dense_table,
                                        uint32_t* state_count, uint32_t** out_offsets,
                                        glop_output** out_flat) {
  try {
    logtrawl::RuleSet rs;
    for (uint32_t i = 0; i < k; ++i) {
      logtrawl::Pattern p;
      p.id = i;
      p.bytes.assign(reinterpret_cast<const char*>(bytes) + off[i], off[i + 1] - off[i]);
      rs.max_len = std::max(rs.max_len, p.bytes.size());
      rs.patterns.push_back(std::move(p));
    }
    const logtrawl::Automaton a = logtrawl::build_failureless_trie(
        logtrawl::truncate_prefixes(rs, prefix_len), logtrawl::Backend::dense, max_states);
    const size_t q = a.state_count;
    auto* d = static_cast<int32_t*>(malloc(q * 256 * 4));
    auto* o = static_cast<uint32_t*>(malloc((q + 1) * 4));
    auto* f = static_cast<glop_output*>(malloc(std::max<size_t>(a.out_flat.size(), 1) * sizeof(glop_output)));
    if (!d || !o || !f) {
      free(d), free(o), free(f);
      return fail(GLOP_ENOMEM, "glop_build_failureless_trie: host allocation");
    }
    memcpy(d, a.dense_table.data(), q * 256 * 4);
    memcpy(o, a.out_offsets.data(), (q + 1) * 4);
    if (!a.out_flat.empty()) memcpy(f, a.out_flat.data(), a.out_flat.size() * sizeof(glop_output));
    *dense_table = d;
    *state_count = (uint32_t)q;
    *out_offsets = o;
    *out_flat = f;
    return GLOP_OK;
  } catch (const logtrawl::CapacityError& e) {
    return fail(GLOP_ECAPACITY, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(GLOP_EINVAL, e.what());
  } catch (const std::bad_alloc&) {
    return fail(GLOP_ENOMEM, "glop_build_failureless_trie: out of memory");
  }
}

void glop_free(void* p) { free(p); }

glop_status glop_last_kernel_ms(glop_ctx* c, float* ms) {
  if (!c || !ms) return fail(GLOP_EINVAL, "glop_last_kernel_ms: null argument");
  if (!c->timed) return fail(GLOP_EINVAL, "glop_last_kernel_ms: no kernel timed yet");
  Dev g(c->device);
  CU(cudaEventSynchronize(c->ev1));
  CU(cudaEventElapsedTime(ms, c->ev0, c->ev1));
  return GLOP_OK;
}

uint64_t glop_ctx_launch_count(glop_ctx* c) { return c ? c->launches : 0; }

// ---- peer exchange (CUDA IPC + copy engines), glop.h
static_assert(sizeof(cudaIpcMemHandle_t) == 64 && sizeof(cudaIpcEventHandle_t) == 64, "64-byte IPC handles");

glop_status glop_peer_alloc(glop_ctx* c, uint64_t bytes, void** d_ptr, void* handle64) {
  if (!c || !d_ptr || !handle64) return fail(GLOP_EINVAL, "glop_peer_alloc: null argument");
  Dev g(c->device);
  *d_ptr = nullptr;
  if (cudaMalloc(d_ptr, std::max<uint64_t>(bytes, 16)) != cudaSuccess) {
    cudaGetLastError();
    return fail(GLOP_ENOMEM, "glop_peer_alloc: cudaMalloc");
  }
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, *d_ptr);
  if (e != cudaSuccess) {
    cudaFree(*d_ptr);
    *d_ptr = nullptr;
    return fail(GLOP_ECUDA, std::string("glop_peer_alloc: ") + cudaGetErrorString(e));
  }
  memcpy(handle64, &h, 64);
  return GLOP_OK;
}

glop_status glop_peer_free(glop_ctx* c, void* d_ptr) {
  if (!c) return fail(GLOP_EINVAL, "glop_peer_free: null context");
  Dev g(c->device);
  if (d_ptr) CU(cudaFree(d_ptr));
  return GLOP_OK;
}

glop_status glop_peer_open(glop_ctx* c, const void* handle64, void** d_ptr) {
  if (!c || !handle64 || !d_ptr) return fail(GLOP_EINVAL, "glop_peer_open: null argument");
  Dev g(c->device);
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  CU(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return GLOP_OK;
}

glop_status glop_peer_close(glop_ctx* c, void* d_ptr) {
  if (!c) return fail(GLOP_EINVAL, "glop_peer_close: null context");
  Dev g(c->device);
  if (d_ptr) CU(cudaIpcCloseMemHandle(d_ptr));
  return GLOP_OK;
}

glop_status glop_peer_event(glop_ctx* c, void** event, void* handle64) {
  if (!c || !event || !handle64) return fail(GLOP_EINVAL, "glop_peer_event: null argument");
  Dev g(c->device);
  cudaEvent_t ev;
  CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming | cudaEventInterprocess));
  cudaIpcEventHandle_t h;
  const cudaError_t e = cudaIpcGetEventHandle(&h, ev);
  if (e != cudaSuccess) {
    cudaEventDestroy(ev);
    return fail(GLOP_ECUDA, std::string("glop_peer_event: ") + cudaGetErrorString(e));
  }
  memcpy(handle64, &h, 64);
  *event = ev;
  return GLOP_OK;
}

glop_status glop_peer_event_open(glop_ctx* c, const void* handle64, void** event) {
  if (!c || !handle64 || !event) return fail(GLOP_EINVAL, "glop_peer_event_open: null argument");
  Dev g(c->device);
  cudaIpcEventHandle_t h;
  memcpy(&h, handle64, 64);
  cudaEvent_t ev;
  CU(cudaIpcOpenEventHandle(&ev, h));
  *event = ev;
  return GLOP_OK;
}

glop_status glop_peer_event_destroy(glop_ctx* c, void* event) {
  if (!c) return fail(GLOP_EINVAL, "glop_peer_event_destroy: null context");
  Dev g(c->device);
  if (event) CU(cudaEventDestroy(static_cast<cudaEvent_t>(event)));
  return GLOP_OK;
}

glop_status glop_peer_record(glop_ctx* c, void* event, void* stream) {
  if (!c || !event) return fail(GLOP_EINVAL, "glop_peer_record: null argument");
  Dev g(c->device);
  CU(cudaEventRecord(static_cast<cudaEvent_t>(event), static_cast<cudaStream_t>(stream)));
  return GLOP_OK;
}

glop_status glop_peer_wait(glop_ctx* c, void* stream, void* event) {
  if (!c || !event) return fail(GLOP_EINVAL, "glop_peer_wait: null argument");
  Dev g(c->device);
  CU(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), static_cast<cudaEvent_t>(event), 0));
  return GLOP_OK;
}

glop_status glop_peer_copy(glop_ctx* c, void* dst, const void* src, uint64_t bytes, void* stream) {
  if (!c || (bytes && (!dst || !src))) return fail(GLOP_EINVAL, "glop_peer_copy: null argument");
  if (!bytes) return GLOP_OK;
  Dev g(c->device);
  CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)));
  return GLOP_OK;
}
uint64_t glop_ctx_fallback_count(glop_ctx* c) { return c ? c->fallbacks : 0; }

glop_status glop_run_pfac_pipeline(glop_ctx* c, const glop_trie* t, const glop_rules* r, const uint8_t* text,
                                   uint64_t n, int text_on_device, glop_alert** alerts, uint64_t* n_alerts,
                                   uint64_t* counts, uint64_t* stage1_hits) {
  return glop_run_pfac_pipeline_shard(c, t, r, text, n, n, 0, text_on_device, alerts, n_alerts, counts,
                                      stage1_hits);
}

glop_status glop_run_pfac_pipeline_shard(glop_ctx* c, const glop_trie* t, const glop_rules* r,
                                         const uint8_t* text, uint64_t n, uint64_t own, uint64_t base,
                                         int text_on_device, glop_alert** alerts, uint64_t* n_alerts,
                                         uint64_t* counts, uint64_t* stage1_hits) {
  return pipeline_host(c, t, r, text, n, own, base, text_on_device, alerts, n_alerts, counts, stage1_hits, nullptr,
                       nullptr);
}

glop_status glop_run_pfac_pipeline_lines(glop_ctx* c, const glop_trie* t, const glop_rules* r, const uint8_t* text,
                                         uint64_t n, int text_on_device, glop_alert** alerts, uint64_t* n_alerts,
                                         uint64_t* counts, uint64_t* stage1_hits, uint64_t** lines,
                                         uint64_t* line_count) {
  if (!lines || !line_count) return fail(GLOP_EINVAL, "glop_run_pfac_pipeline_lines: null argument");
  return pipeline_host(c, t, r, text, n, n, 0, text_on_device, alerts, n_alerts, counts, stage1_hits, lines,
                       line_count);
}

glop_status glop_run_pfac_pipeline_shard_lines(glop_ctx* c, const glop_trie* t, const glop_rules* r,
                                               const uint8_t* text, uint64_t n, uint64_t own, uint64_t base,
                                               int text_on_device, glop_alert** alerts, uint64_t* n_alerts,
                                               uint64_t* counts, uint64_t* stage1_hits, uint64_t** lines,
                                               uint64_t* line_count) {
  if (!lines || !line_count) return fail(GLOP_EINVAL, "glop_run_pfac_pipeline_shard_lines: null argument");
  return pipeline_host(c, t, r, text, n, own, base, text_on_device, alerts, n_alerts, counts, stage1_hits, lines,
                       line_count);
}

// ---- streaming: the text arrives in caller buffers of any size; windows of
// W bytes are scanned as they fill, each reading max(depth, max_len) - 1 bytes
// of the next one (carried over), so a match straddling two feed() calls or
// two windows is found exactly once (SPEC.md:290 windowing).
struct glop_stream {
  glop_ctx* c = nullptr;
  const glop_trie* t = nullptr;
  const glop_rules* r = nullptr;
  uint64_t halo = 0, W = 0, fill = 0, pos = 0;
  void* pin = nullptr;  // window staging (pinned): bytes [pos, pos + fill) of the text
  DBuf dtext;
  Accum A;
  glop_status err = GLOP_OK;
};

namespace {
glop_status stream_window(glop_stream* st, uint64_t own) {
  glop_ctx* c = st->c;
  CU(cudaMemcpyAsync(st->dtext.p, st->pin, st->fill, cudaMemcpyHostToDevice, c->stream));
  return accum_window(c, st->t, st->r, st->A, st->dtext.as<uint8_t>(), st->fill, own, st->pos);
}
}  // namespace

glop_status glop_stream_begin(glop_ctx* c, const glop_trie* t, const glop_rules* r, int with_lines,
                              glop_stream** out) {
  if (!c || !t || !r || !out) return fail(GLOP_EINVAL, "glop_stream_begin: null argument");
  *out = nullptr;
  std::lock_guard<std::mutex> lk(c->mu);
  Dev g(c->device);
  auto* st = new glop_stream();
  st->c = c;
  st->t = t;
  st->r = r;
  st->halo = std::max<uint64_t>(std::max<uint64_t>(t->info.max_depth, r->max_len), 1) - 1;
  const char* env = getenv("GLOP_STREAM_WINDOW");  // tests: small windows
  st->W = std::max<uint64_t>(env ? strtoull(env, nullptr, 10) : kStreamChunk, st->halo + 1);
  glop_status s = GLOP_OK;
  if (cudaMallocHost(&st->pin, st->W + st->halo + 64) != cudaSuccess) s = fail(GLOP_ENOMEM, "glop_stream_begin: pinned buffer");
  if (s == GLOP_OK) s = st->dtext.ensure(st->W + st->halo + 64);
  if (s == GLOP_OK) s = accum_begin(c, st->A, r->view.n_patterns, with_lines != 0);
  if (s != GLOP_OK) {
    if (st->pin) cudaFreeHost(st->pin);
    st->dtext.release();
    st->A.release();
    delete st;
    return s;
  }
  *out = st;
  return GLOP_OK;
}

glop_status glop_stream_feed(glop_stream* st, const uint8_t* data, uint64_t len) {
  if (!st || (len && !data)) return fail(GLOP_EINVAL, "glop_stream_feed: null argument");
  if (st->err != GLOP_OK) return fail(st->err, "glop_stream_feed: the stream failed earlier");
  std::lock_guard<std::mutex> lk(st->c->mu);
  Dev g(st->c->device);
  const uint64_t full = st->W + st->halo;
  while (len) {
    const uint64_t take = std::min<uint64_t>(len, full - st->fill);
    parallel_memcpy(static_cast<uint8_t*>(st->pin) + st->fill, data, take);
    st->fill += take;
    data += take;
    len -= take;
    if (st->fill == full) {  // window [pos, pos + W) with its halo: scan, then carry the halo
      const glop_status s = stream_window(st, st->W);
      if (s != GLOP_OK) return st->err = s;
      memmove(st->pin, static_cast<uint8_t*>(st->pin) + st->W, st->halo);  // (the copy above has completed)
      st->fill = st->halo;
      st->pos += st->W;
    }
  }
  return GLOP_OK;
}

glop_status glop_stream_end(glop_stream* st, glop_alert** alerts, uint64_t* n_alerts, uint64_t* counts,
                            uint64_t* stage1_hits, uint64_t** lines, uint64_t* line_count, uint64_t* bytes) {
  if (!st) return fail(GLOP_EINVAL, "glop_stream_end: null stream");
  glop_status s = st->err;
  {
    std::lock_guard<std::mutex> lk(st->c->mu);
    Dev g(st->c->device);
    if (s == GLOP_OK && (!alerts || !n_alerts)) s = fail(GLOP_EINVAL, "glop_stream_end: null argument");
    if (s == GLOP_OK && st->fill) s = stream_window(st, st->fill);  // the tail owns every remaining start
    if (s == GLOP_OK)
      s = accum_end(st->c, st->A, alerts, n_alerts, counts, stage1_hits, lines, line_count);
    if (s == GLOP_OK && bytes) *bytes = st->pos + st->fill;
    cudaStreamSynchronize(st->c->stream);
    st->dtext.release();
    st->A.release();
  }
  if (st->pin) cudaFreeHost(st->pin);
  delete st;
  return s;
}

glop_status glop_chunked_ac_scan(glop_ctx* c, const glop_trie* t, const uint8_t* text, uint64_t n,
                                 int text_on_device, uint64_t chunk_size, uint64_t overlap, glop_hit** matches,
                                 uint64_t* n_matches) {
  if (!c || !t || !matches || !n_matches) return fail(GLOP_EINVAL, "glop_chunked_ac_scan: null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  Dev g(c->device);
  *matches = nullptr;
  *n_matches = 0;
  const uint8_t* d_text = nullptr;
  TRY(to_device_text(c, text, n, text_on_device, &d_text));
  uint64_t cap = std::max<uint64_t>(1 << 16, c->out.bytes / sizeof(glop_hit));
  TRY(c->out.ensure(cap * sizeof(glop_hit)));
  uint64_t total = 0;
  glop_status s = chunked_ac_impl(c, t, d_text, n, chunk_size, overlap, c->out.as<glop_hit>(), cap, &total);
  if (s == GLOP_ECAPACITY && total > cap) {
    c->out.release();
    cap = total;
    TRY(c->out.ensure(cap * sizeof(glop_hit)));
    s = chunked_ac_impl(c, t, d_text, n, chunk_size, overlap, c->out.as<glop_hit>(), cap, &total);
  }
  if (s != GLOP_OK) return s;
  glop_hit* h = static_cast<glop_hit*>(malloc(std::max<uint64_t>(total, 1) * sizeof(glop_hit)));
  if (!h) return fail(GLOP_ENOMEM, "glop_chunked_ac_scan: host allocation");
  cudaError_t e = cudaSuccess;
  if (total) e = cudaMemcpyAsync(h, c->out.p, total * sizeof(glop_hit), cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    free(h);
    return fail(GLOP_ECUDA, cudaGetErrorString(e));
  }
  *matches = h;
  *n_matches = total;
  return GLOP_OK;
}

}  // extern "C"

namespace {
glop_status pipeline_host(glop_ctx* c, const glop_trie* t, const glop_rules* r, const uint8_t* text, uint64_t n,
                          uint64_t own, uint64_t base, int text_on_device, glop_alert** alerts, uint64_t* n_alerts,
                          uint64_t* counts, uint64_t* stage1_hits, uint64_t** lines, uint64_t* line_count) {
  if (!c || !t || !r || !alerts || !n_alerts) return fail(GLOP_EINVAL, "glop_run_pfac_pipeline: null argument");
  if (own > n) return fail(GLOP_EINVAL, "glop_run_pfac_pipeline: own > n");
  std::lock_guard<std::mutex> lk(c->mu);
  Dev g(c->device);
  *alerts = nullptr;
  *n_alerts = 0;
  if (!text_on_device && own > kStreamChunk)
    return run_pipeline_streamed(c, t, r, text, n, own, base, alerts, n_alerts, counts, stage1_hits, lines,
                                 line_count);
  const uint8_t* d_text = nullptr;
  TRY(to_device_text(c, text, n, text_on_device, &d_text));
  const uint32_t k = r->view.n_patterns;
  TRY(c->spill.ensure((size_t)(k + 1) * 8));
  uint64_t* d_counts = c->spill.as<uint64_t>();
  TRY(c->palerts.ensure(std::max<size_t>(c->palerts.bytes, (1 << 16) * sizeof(glop_alert))));
  uint64_t nh = 0, kept = 0, acap = c->palerts.bytes / sizeof(glop_alert);
  glop_status s = pipeline_device_impl(c, t, r, d_text, n, own, base, nullptr, 0, c->palerts.as<glop_alert>(), acap,
                                       d_counts, &nh, &kept);
  if (s == GLOP_ECAPACITY && kept > acap) {
    c->palerts.release();
    TRY(c->palerts.ensure(kept * sizeof(glop_alert)));
    s = pipeline_device_impl(c, t, r, d_text, n, own, base, nullptr, 0, c->palerts.as<glop_alert>(), kept, d_counts,
                             &nh, &kept);
  }
  if (s != GLOP_OK) return s;
  if (stage1_hits) *stage1_hits = nh;
  uint64_t* d_lf = nullptr;
  if (lines || line_count) {  // LineIndex over the owned bytes [0, own), on the device
    TRY(c->plines.ensure(kept * 8 + 16));
    d_lf = c->plines.as<uint64_t>() + kept + 1;
    CU(cudaMemsetAsync(d_lf, 0, 8, c->stream));
    TRY(line_numbers_impl(c, d_text, own, base, c->palerts.p, sizeof(glop_alert), kept, c->plines.as<uint64_t>(),
                          nullptr, d_lf));
  }
  TRY(alerts_to_host(c, c->palerts.as<glop_alert>(), kept, d_counts, k, counts, alerts, c->plines.as<uint64_t>(),
                     lines, d_lf, line_count));
  *n_alerts = kept;
  return GLOP_OK;
}
}  // namespace

extern "C" {

glop_status glop_run_pfac_pipeline_device_async(glop_ctx* c, const glop_trie* t, const glop_rules* r,
                                                const uint8_t* d_text, uint64_t n, uint64_t own, uint64_t base,
                                                glop_hit* d_hits, uint64_t hit_cap, glop_alert* d_alerts,
                                                uint64_t alert_cap, uint64_t* d_counts,
                                                glop_pipeline_ticket* ticket) {
  if (!c || !t || !r || !ticket || (!d_alerts && alert_cap))
    return fail(GLOP_EINVAL, "glop_run_pfac_pipeline_device_async: null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  Dev g(c->device);
  uint64_t nh = 0, na = 0;
  memset(ticket, 0, sizeof *ticket);
  const glop_status s = pipeline_device_impl(c, t, r, d_text, n, own, base, d_hits, hit_cap, d_alerts, alert_cap,
                                             d_counts, &nh, &na, ticket);
  if (s != GLOP_OK || ticket->region == 0) {
    // failed, or the general path ran synchronously: the ticket holds the outcome
    ticket->done = s == GLOP_OK ? 1 : 2;
    ticket->raw[0] = nh;
    ticket->raw[5] = na;
    ticket->raw[7] = (uint64_t)s;
  }
  return s;
}

glop_status glop_pipeline_ticket_result(const glop_pipeline_ticket* k, uint64_t* n_hits, uint64_t* n_alerts) {
  if (!k || !n_hits || !n_alerts) return fail(GLOP_EINVAL, "glop_pipeline_ticket_result: null argument");
  if (k->done == 1) {  // completed synchronously
    *n_hits = k->raw[0];
    *n_alerts = k->raw[5];
    return GLOP_OK;
  }
  if (k->done == 2) return fail((glop_status)k->raw[7], "run_pfac_pipeline: failed");
  const uint64_t* h = k->raw;
  if ((h[kStFlags] & 1u) || h[kStMaxRegion] > k->region)
    return fail(GLOP_EAGAIN, "run_pfac_pipeline: this input needs the synchronous path (hit buffer / staging overflow)");
  if (h[kStVerify] & 1u) return fail(GLOP_ELOGIC, "verify_hits: hit extends past end of text");
  *n_hits = h[kStTotal];
  *n_alerts = k->stage2 ? h[kStKept] : h[kStTotal];
  if (*n_hits > k->hit_cap || *n_alerts > k->alert_cap) return fail(GLOP_ECAPACITY, "run_pfac_pipeline: output capacity");
  return GLOP_OK;
}

glop_status glop_run_pfac_pipeline_device(glop_ctx* c, const glop_trie* t, const glop_rules* r,
                                          const uint8_t* d_text, uint64_t n, uint64_t own, uint64_t base,
                                          glop_hit* d_hits, uint64_t hit_cap, glop_alert* d_alerts,
                                          uint64_t alert_cap, uint64_t* d_counts, uint64_t* n_hits,
                                          uint64_t* n_alerts) {
  if (!c || !t || !r || !n_hits || !n_alerts || (!d_alerts && alert_cap))
    return fail(GLOP_EINVAL, "glop_run_pfac_pipeline_device: null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  Dev g(c->device);
  return pipeline_device_impl(c, t, r, d_text, n, own, base, d_hits, hit_cap, d_alerts, alert_cap, d_counts, n_hits,
                              n_alerts);
}

glop_status glop_line_numbers_device(glop_ctx* c, const uint8_t* d_text, uint64_t n, uint64_t base,
                                     const void* d_records, uint32_t stride, uint64_t count, uint64_t* d_lines) {
  if (!c || (count && (!d_text || !d_records || !d_lines)) || stride < 8)
    return fail(GLOP_EINVAL, "glop_line_numbers_device: bad argument");
  std::lock_guard<std::mutex> lk(c->mu);
  Dev g(c->device);
  return line_numbers_impl(c, d_text, n, base, d_records, stride, count, d_lines, nullptr, nullptr);
}

glop_status glop_line_numbers(glop_ctx* c, const uint8_t* text, uint64_t n, int text_on_device,
                              const uint64_t* offsets, uint64_t count, uint64_t* lines) {
  if (!c || (count && (!offsets || !lines))) return fail(GLOP_EINVAL, "glop_line_numbers: null argument");
  for (uint64_t i = 0; i < count; ++i)
    if (offsets[i] > n) return fail(GLOP_EINVAL, "glop_line_numbers: offset past the end of text");
  std::lock_guard<std::mutex> lk(c->mu);
  Dev g(c->device);
  if (count == 0) return GLOP_OK;
  const uint8_t* d_text = nullptr;
  TRY(to_device_text(c, text, n, text_on_device, &d_text));
  TRY(c->loffs.ensure(count * 16));
  uint64_t* d_offs = c->loffs.as<uint64_t>();
  CU(cudaMemcpyAsync(d_offs, offsets, count * 8, cudaMemcpyHostToDevice, c->stream));
  TRY(line_numbers_impl(c, d_text, n, 0, d_offs, 8, count, d_offs + count, nullptr, nullptr));
  CU(cudaMemcpyAsync(lines, d_offs + count, count * 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return GLOP_OK;
}

glop_status glop_device_alloc(glop_ctx* c, uint64_t bytes, void** out) {
  Dev g(c->device);
  CU(cudaMalloc(out, std::max<uint64_t>(bytes, 16)));
  return GLOP_OK;
}
glop_status glop_device_free(glop_ctx* c, void* p) {
  Dev g(c->device);
  CU(cudaFree(p));
  return GLOP_OK;
}
glop_status glop_host_alloc(uint64_t bytes, void** out) {
  CU(cudaMallocHost(out, std::max<uint64_t>(bytes, 16)));
  return GLOP_OK;
}
glop_status glop_host_free(void* p) {
  CU(cudaFreeHost(p));
  return GLOP_OK;
}
glop_status glop_memcpy(glop_ctx* c, void* dst, const void* src, uint64_t bytes, int kind) {
  Dev g(c->device);
  cudaMemcpyKind k = kind == 1 ? cudaMemcpyHostToDevice
                               : (kind == 2 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice);
  CU(cudaMemcpyAsync(dst, src, bytes, k, c->stream));
  return GLOP_OK;
}

glop_status glop_gen_syslog_device(glop_ctx* c, uint8_t* d_out, uint64_t begin, uint64_t n, uint64_t seed) {
  if (n == 0) return GLOP_OK;
  Dev g(c->device);
  const uint64_t blocks = (begin + n - 1) / glop_corpus::kBlock - begin / glop_corpus::kBlock + 1;
  const uint32_t grid = (uint32_t)std::min<uint64_t>((blocks + 127) / 128, 65535);
  ++c->launches;
  gen_syslog_kernel<<<grid, 128, 0, c->stream>>>(d_out, begin, n, seed);
  CU(cudaGetLastError());
  return GLOP_OK;
}

glop_status glop_gen_syslog_host(uint8_t* out, uint64_t begin, uint64_t n, uint64_t seed, unsigned threads) {
  glop_workload::gen_syslog(out, begin, n, seed, threads);
  return GLOP_OK;
}

glop_status glop_gen_payload_device(glop_ctx* c, uint8_t* d_out, uint64_t begin, uint64_t n, uint64_t seed) {
  if (n == 0) return GLOP_OK;
  Dev g(c->device);
  const uint64_t blocks = (begin + n - 1) / glop_payload::kBlock - begin / glop_payload::kBlock + 1;
  const uint32_t grid = (uint32_t)std::min<uint64_t>((blocks + 127) / 128, 65535);
  ++c->launches;
  gen_payload_kernel<<<grid, 128, 0, c->stream>>>(d_out, begin, n, seed);
  CU(cudaGetLastError());
  return GLOP_OK;
}

glop_status glop_gen_payload_host(uint8_t* out, uint64_t begin, uint64_t n, uint64_t seed, unsigned threads) {
  glop_workload::gen_payload(out, begin, n, seed, threads);
  return GLOP_OK;
}

glop_status glop_gen_dpi_rules(uint32_t k, uint32_t seed, uint32_t min_len, uint32_t max_len, uint8_t* bytes,
                               uint64_t* off) {
  if (min_len < 1 || max_len < min_len) return fail(GLOP_EINVAL, "glop_gen_dpi_rules: bad lengths");
  const auto rules = glop_workload::dpi_rules(k, seed, min_len, max_len);
  uint64_t o = 0;
  for (uint32_t i = 0; i < k; ++i) {
    off[i] = o;
    memcpy(bytes + o, rules[i].data(), rules[i].size());
    o += rules[i].size();
  }
  off[k] = o;
  return GLOP_OK;
}

glop_status glop_gen_reference_log(uint8_t* out, uint64_t size, uint32_t seed, uint64_t line_len) {
  if (size == 0 || line_len < 2) return fail(GLOP_EINVAL, "generate_log: bad size/line_len");
  std::string s = glop_workload::reference_generate_log(size, seed, line_len);
  memcpy(out, s.data(), size);
  return GLOP_OK;
}

glop_status glop_gen_rules(uint32_t k, uint32_t seed, uint32_t len, uint8_t* bytes, uint8_t* is_vocab) {
  auto rules = glop_workload::synthetic_rules(k, seed, len);
  for (uint32_t i = 0; i < k; ++i) {
    memcpy(bytes + (size_t)i * len, rules[i].bytes.data(), len);
    if (is_vocab) is_vocab[i] = rules[i].name.rfind("vocab-", 0) == 0;
  }
  return GLOP_OK;
}

}  // extern "C"

#include "group.inl"
