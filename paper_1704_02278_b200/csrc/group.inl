// group.cpp -- multi-GPU inside libglop: a glop_group is one
// glop_ctx per member device (a device may repeat: N contexts on one GPU are
// how a one-GPU box exercises the N-way split).  A group call splits the text
// into contiguous shards, member g owning starts [lo_g, lo_g + own_g) and
// reading a halo past them (the ownership rule of scan.hpp:230-232; the
// contiguous split of detail::parallel_ranges, scan.hpp:59-79), runs every
// member's shard on its own host thread and its own CUDA stream, and merges:
// rank-order concatenation of the per-shard results is already sorted
// (owned ranges ascend and are disjoint), per-pattern counts add up, and
// line numbers / KMP comparison counts are offset by the shards before.
//
// The merge target is host memory (the API returns host arrays), so each
// member copies its own alerts straight to the host over its own PCIe link;
// a collective to one GPU first would only add a hop.  Cross-process runs
// (torchrun, one process per GPU) use the per-rank shard calls plus NCCL
// (paper_1704_02278_b200/shards.py, bench.py).
//
// Host-only composition of the single-context C ABI (glop.h); no kernels.
// Included by glop.cu (shares its per-thread error message).

struct glop_group {
  std::vector<int> devices;
  std::vector<glop_ctx*> ctx;
  uint64_t min_shard = 64ull << 20;  // below this many bytes per member, fewer members work
};

struct glop_group_trie {
  std::vector<glop_trie*> member;  // per member (shared by members on one device)
  std::vector<glop_trie*> owned;
  uint32_t max_depth = 0;
};

struct glop_group_rules {
  std::vector<glop_rules*> member;
  std::vector<glop_rules*> owned;
  uint64_t max_len = 0;
};

namespace {

glop_status gfail(glop_status s, const std::string& msg) { return fail(s, msg); }

// Runs fn(member) for members [0, parts) on one host thread each; returns the
// first failure (with its message, which glop_last_error keeps per thread).
template <typename Fn>
glop_status run_members(int parts, Fn&& fn) {
  std::vector<glop_status> st(parts, GLOP_OK);
  std::vector<std::string> err(parts);
  auto body = [&](int g) {
    st[g] = fn(g);
    if (st[g] != GLOP_OK) err[g] = glop_last_error();
  };
  if (parts == 1) {
    body(0);
  } else {
    std::vector<std::thread> pool;
    for (int g = 1; g < parts; ++g) pool.emplace_back(body, g);
    body(0);
    for (auto& t : pool) t.join();
  }
  for (int g = 0; g < parts; ++g)
    if (st[g] != GLOP_OK) return gfail(st[g], err[g]);
  return GLOP_OK;
}

struct Shard {
  uint64_t lo, own, read;
};

std::vector<Shard> plan(const glop_group* g, uint64_t n, uint64_t halo) {
  const uint64_t members = g->ctx.size();
  uint64_t parts = std::min<uint64_t>(members, std::max<uint64_t>(1, n / std::max<uint64_t>(g->min_shard, 1)));
  parts = std::max<uint64_t>(parts, 1);
  std::vector<uint64_t> lo(parts), own(parts), rd(parts);
  glop_plan_shards(n, (uint32_t)parts, halo, lo.data(), own.data(), rd.data());
  std::vector<Shard> out(parts);
  for (uint64_t i = 0; i < parts; ++i) out[i] = Shard{lo[i], own[i], rd[i]};
  return out;
}

template <typename T>
glop_status concat(const std::vector<T*>& parts, const std::vector<uint64_t>& sizes, T** out, uint64_t* total) {
  uint64_t n = 0;
  for (uint64_t s : sizes) n += s;
  T* all = static_cast<T*>(malloc(std::max<uint64_t>(n, 1) * sizeof(T)));
  if (!all) return gfail(GLOP_ENOMEM, "glop_group: host allocation");
  uint64_t at = 0;
  for (size_t i = 0; i < parts.size(); ++i) {
    if (sizes[i]) memcpy(all + at, parts[i], sizes[i] * sizeof(T));
    at += sizes[i];
  }
  *out = all;
  *total = n;
  return GLOP_OK;
}

void free_all(std::vector<void*> ps) {
  for (void* p : ps) glop_free(p);
}

}  // namespace

extern "C" {

glop_status glop_plan_shards(uint64_t n, uint32_t parts, uint64_t halo, uint64_t* lo, uint64_t* own,
                             uint64_t* read) {
  if (parts == 0 || !lo || !own || !read) return gfail(GLOP_EINVAL, "glop_plan_shards: bad argument");
  const uint64_t per = n / parts, extra = n % parts;
  uint64_t at = 0;
  for (uint32_t g = 0; g < parts; ++g) {
    lo[g] = at;
    own[g] = per + (g < extra ? 1 : 0);
    read[g] = std::min<uint64_t>(own[g] + halo, n - at);
    at += own[g];
  }
  return GLOP_OK;
}

glop_status glop_group_create(const int* devices, int n_devices, glop_group** out) {
  *out = nullptr;
  std::vector<int> devs;
  if (devices) {
    if (n_devices < 1) return gfail(GLOP_EINVAL, "glop_group_create: no devices");
    devs.assign(devices, devices + n_devices);
  } else {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count < 1) {
      cudaGetLastError();
      return gfail(GLOP_ECUDA, "glop_group_create: no CUDA device");
    }
    const int want = n_devices > 0 ? std::min(n_devices, count) : count;
    for (int d = 0; d < want; ++d) devs.push_back(d);
  }
  auto* g = new glop_group();
  g->devices = devs;
  if (const char* env = getenv("GLOP_GROUP_MIN_SHARD")) g->min_shard = std::max<uint64_t>(1, strtoull(env, nullptr, 10));
  for (int d : devs) {
    glop_ctx* c = nullptr;
    const glop_status s = glop_ctx_create(d, &c);
    if (s != GLOP_OK) {
      const std::string msg = glop_last_error();
      glop_group_destroy(g);
      return gfail(s, msg);
    }
    g->ctx.push_back(c);
  }
  *out = g;
  return GLOP_OK;
}

glop_status glop_group_destroy(glop_group* g) {
  if (!g) return GLOP_OK;
  for (glop_ctx* c : g->ctx) glop_ctx_destroy(c);
  delete g;
  return GLOP_OK;
}

int glop_group_size(const glop_group* g) { return g ? (int)g->ctx.size() : 0; }

glop_ctx* glop_group_ctx(glop_group* g, int member) {
  return g && member >= 0 && member < (int)g->ctx.size() ? g->ctx[member] : nullptr;
}

glop_status glop_group_trie_upload(glop_group* g, const int32_t* dense, uint32_t Q, const uint32_t* out_offsets,
                                   const glop_output* out_flat, glop_group_trie** out) {
  *out = nullptr;
  if (!g) return gfail(GLOP_EINVAL, "glop_group_trie_upload: null group");
  auto* t = new glop_group_trie();
  t->member.assign(g->ctx.size(), nullptr);
  for (size_t i = 0; i < g->ctx.size(); ++i) {
    for (size_t j = 0; j < i; ++j)
      if (g->devices[j] == g->devices[i]) t->member[i] = t->member[j];
    if (t->member[i]) continue;
    glop_trie* x = nullptr;
    const glop_status s = glop_trie_upload(g->ctx[i], dense, Q, out_offsets, out_flat, &x);
    if (s != GLOP_OK) {
      const std::string msg = glop_last_error();
      glop_group_trie_destroy(t);
      return gfail(s, msg);
    }
    t->member[i] = x;
    t->owned.push_back(x);
  }
  glop_trie_info info{};
  glop_trie_get_info(t->member[0], &info);
  t->max_depth = info.max_depth;
  *out = t;
  return GLOP_OK;
}

glop_trie* glop_group_trie_member(glop_group_trie* t, int member) {
  return t && member >= 0 && member < (int)t->member.size() ? t->member[member] : nullptr;
}

glop_status glop_group_trie_destroy(glop_group_trie* t) {
  if (!t) return GLOP_OK;
  for (glop_trie* x : t->owned) glop_trie_destroy(x);
  delete t;
  return GLOP_OK;
}

glop_status glop_group_rules_upload(glop_group* g, const uint8_t* bytes, const uint64_t* off, uint32_t n_patterns,
                                    uint64_t prefix_len, glop_group_rules** out) {
  *out = nullptr;
  if (!g || !off) return gfail(GLOP_EINVAL, "glop_group_rules_upload: null argument");
  auto* r = new glop_group_rules();
  r->member.assign(g->ctx.size(), nullptr);
  for (uint32_t i = 0; i < n_patterns; ++i) r->max_len = std::max<uint64_t>(r->max_len, off[i + 1] - off[i]);
  for (size_t i = 0; i < g->ctx.size(); ++i) {
    for (size_t j = 0; j < i; ++j)
      if (g->devices[j] == g->devices[i]) r->member[i] = r->member[j];
    if (r->member[i]) continue;
    glop_rules* x = nullptr;
    const glop_status s = glop_rules_upload(g->ctx[i], bytes, off, n_patterns, prefix_len, &x);
    if (s != GLOP_OK) {
      const std::string msg = glop_last_error();
      glop_group_rules_destroy(r);
      return gfail(s, msg);
    }
    r->member[i] = x;
    r->owned.push_back(x);
  }
  *out = r;
  return GLOP_OK;
}

glop_rules* glop_group_rules_member(glop_group_rules* r, int member) {
  return r && member >= 0 && member < (int)r->member.size() ? r->member[member] : nullptr;
}

glop_status glop_group_rules_destroy(glop_group_rules* r) {
  if (!r) return GLOP_OK;
  for (glop_rules* x : r->owned) glop_rules_destroy(x);
  delete r;
  return GLOP_OK;
}

glop_status glop_group_pfac_scan(glop_group* g, const glop_group_trie* t, const uint8_t* text, uint64_t n,
                                 glop_hit** hits, uint64_t* n_hits) {
  if (!g || !t || !hits || !n_hits) return gfail(GLOP_EINVAL, "glop_group_pfac_scan: null argument");
  *hits = nullptr;
  *n_hits = 0;
  const std::vector<Shard> sh = plan(g, n, t->max_depth ? t->max_depth - 1 : 0);
  const int parts = (int)sh.size();
  std::vector<glop_hit*> part(parts, nullptr);
  std::vector<uint64_t> cnt(parts, 0);
  glop_status s = run_members(parts, [&](int m) {
    return glop_pfac_scan_shard(g->ctx[m], t->member[m], text + sh[m].lo, sh[m].read, sh[m].own, sh[m].lo, 0,
                                &part[m], &cnt[m]);
  });
  if (s == GLOP_OK) s = concat(part, cnt, hits, n_hits);
  free_all(std::vector<void*>(part.begin(), part.end()));
  return s;
}

glop_status glop_group_run_pfac_pipeline(glop_group* g, const glop_group_trie* t, const glop_group_rules* r,
                                         const uint8_t* text, uint64_t n, glop_alert** alerts, uint64_t* n_alerts,
                                         uint64_t* counts, uint64_t* stage1_hits, uint64_t** lines,
                                         uint64_t* line_count) {
  if (!g || !t || !r || !alerts || !n_alerts || (!lines) != (!line_count))
    return gfail(GLOP_EINVAL, "glop_group_run_pfac_pipeline: bad argument");
  *alerts = nullptr;
  *n_alerts = 0;
  const uint64_t halo = std::max<uint64_t>(std::max<uint64_t>(t->max_depth, r->max_len), 1) - 1;
  const std::vector<Shard> sh = plan(g, n, halo);
  const int parts = (int)sh.size();
  std::vector<glop_alert*> part(parts, nullptr);
  std::vector<uint64_t*> plines(parts, nullptr);
  std::vector<uint64_t> cnt(parts, 0), s1(parts, 0), lc(parts, 0);
  std::vector<std::vector<uint64_t>> pc(parts);
  uint64_t nl = 0;
  glop_status s = run_members(parts, [&](int m) {
    pc[m].assign(counts ? r->member[m]->view.n_patterns : 0, 0);
    if (lines)
      return glop_run_pfac_pipeline_shard_lines(g->ctx[m], t->member[m], r->member[m], text + sh[m].lo, sh[m].read,
                                                sh[m].own, sh[m].lo, 0, &part[m], &cnt[m],
                                                counts ? pc[m].data() : nullptr, &s1[m], &plines[m], &lc[m]);
    return glop_run_pfac_pipeline_shard(g->ctx[m], t->member[m], r->member[m], text + sh[m].lo, sh[m].read,
                                        sh[m].own, sh[m].lo, 0, &part[m], &cnt[m], counts ? pc[m].data() : nullptr,
                                        &s1[m]);
  });
  if (s == GLOP_OK) s = concat(part, cnt, alerts, n_alerts);
  if (s == GLOP_OK && lines) {
    // member m's lines count from its shard's start: add the LFs of the shards before it
    s = concat(plines, cnt, lines, &nl);
    uint64_t before = 0, at = 0;
    for (int m = 0; m < parts && s == GLOP_OK; ++m) {
      for (uint64_t i = 0; i < cnt[m]; ++i) (*lines)[at + i] += before;
      at += cnt[m];
      before += lc[m] - 1;  // line_count - 1 = LF bytes in the owned part
    }
    *line_count = before + 1;
  }
  if (s == GLOP_OK) {
    if (counts) {
      const size_t kk = pc[0].size();
      for (size_t i = 0; i < kk; ++i) {
        uint64_t x = 0;
        for (int m = 0; m < parts; ++m) x += pc[m][i];
        counts[i] = x;
      }
    }
    if (stage1_hits) {
      uint64_t x = 0;
      for (uint64_t v : s1) x += v;
      *stage1_hits = x;
    }
  } else {
    glop_free(*alerts);
    *alerts = nullptr;
    *n_alerts = 0;
  }
  free_all(std::vector<void*>(part.begin(), part.end()));
  free_all(std::vector<void*>(plines.begin(), plines.end()));
  return s;
}

glop_status glop_group_kmp_search(glop_group* g, const uint8_t* p, uint32_t m, const uint32_t* failure,
                                  const uint8_t* text, uint64_t n, uint64_t** offsets, uint64_t* n_offsets,
                                  uint64_t* comparisons) {
  if (!g || !offsets || !n_offsets) return gfail(GLOP_EINVAL, "glop_group_kmp_search: null argument");
  *offsets = nullptr;
  *n_offsets = 0;
  // canonical failure tables shard exactly (left context m-1 recovers the
  // state); anything else runs the reference's sequential walk on member 0
  bool canonical = m > 0 && m < 8192;
  for (uint32_t i = 0, kk = 0; i < m && canonical; ++i) {
    if (i > 0) {
      while (kk > 0 && p[i] != p[kk]) kk = failure[kk - 1];
      if (p[i] == p[kk]) ++kk;
    }
    canonical = failure[i] == (i ? kk : 0u);
  }
  const uint64_t halo = m ? m - 1 : 0;
  const std::vector<Shard> sh = canonical ? plan(g, n, halo) : std::vector<Shard>{Shard{0, n, n}};
  const int parts = (int)sh.size();
  std::vector<uint64_t*> part(parts, nullptr);
  std::vector<uint64_t> cnt(parts, 0), cmp(parts, 0);
  glop_status s = run_members(parts, [&](int w) {
    const uint64_t left = std::min<uint64_t>(sh[w].lo, halo);  // context to recover the KMP state
    const uint64_t base = sh[w].lo - left;
    return glop_kmp_search_shard(g->ctx[w], p, m, failure, text + base, left + sh[w].read, left,
                                 left + sh[w].own, base, 0, &part[w], &cnt[w], &cmp[w]);
  });
  if (s == GLOP_OK) s = concat(part, cnt, offsets, n_offsets);
  if (s == GLOP_OK && comparisons)
    for (uint64_t c : cmp) *comparisons += c;
  free_all(std::vector<void*>(part.begin(), part.end()));
  return s;
}

}  // extern "C"

// ---- streaming over the group: the text arrives in pieces; windows of W
// bytes (+ the halo carried from the next window) are handed round-robin to
// the members, each scanning its windows on its own thread, stream and PCIe
// link; the results merge in window order at the end.
struct glop_group_stream {
  glop_group* g = nullptr;
  const glop_group_trie* t = nullptr;
  const glop_group_rules* r = nullptr;
  bool lines = false;
  uint64_t W = 0, halo = 0, pos = 0, fill = 0, windows = 0;
  uint8_t* cur = nullptr;                  // the window being filled (pinned)
  std::vector<uint8_t*> pool;              // free pinned window buffers
  std::vector<uint8_t*> all;               // every buffer (freed at the end)
  struct Result {
    glop_alert* alerts = nullptr;
    uint64_t* lines = nullptr;
    uint64_t n_alerts = 0, stage1 = 0, line_count = 0;
    uint64_t own = 0, read = 0;  // the window: starts owned, bytes read (own + halo)
    std::vector<uint64_t> counts;
    glop_status st = GLOP_OK;
    std::string err;
  };
  std::vector<Result> results;             // by window index
  struct Member {
    std::thread th;
    std::mutex mu;
    std::condition_variable cv;
    std::deque<std::pair<uint64_t, uint8_t*>> q;  // (window index, buffer)
    bool stop = false;
  };
  std::vector<std::unique_ptr<Member>> members;
  std::mutex pool_mu;
  std::condition_variable pool_cv;
  std::mutex res_mu;
};

namespace {
void gs_worker(glop_group_stream* gs, int m) {
  glop_group_stream::Member& mb = *gs->members[m];
  for (;;) {
    std::pair<uint64_t, uint8_t*> job;
    {
      std::unique_lock<std::mutex> lk(mb.mu);
      mb.cv.wait(lk, [&] { return mb.stop || !mb.q.empty(); });
      if (mb.q.empty()) return;
      job = mb.q.front();
      mb.q.pop_front();
    }
    const uint64_t w = job.first, lo = w * gs->W;
    uint64_t own, rd;
    {
      std::lock_guard<std::mutex> lk(gs->res_mu);
      own = gs->results[w].own;
      rd = gs->results[w].read;
    }
    glop_group_stream::Result res;
    res.own = own;
    res.read = rd;
    res.counts.assign(gs->r->member[m]->view.n_patterns, 0);
    glop_status s;
    if (gs->lines)
      s = glop_run_pfac_pipeline_shard_lines(gs->g->ctx[m], gs->t->member[m], gs->r->member[m], job.second, rd, own,
                                             lo, 0, &res.alerts, &res.n_alerts, res.counts.data(), &res.stage1,
                                             &res.lines, &res.line_count);
    else
      s = glop_run_pfac_pipeline_shard(gs->g->ctx[m], gs->t->member[m], gs->r->member[m], job.second, rd, own, lo, 0,
                                       &res.alerts, &res.n_alerts, res.counts.data(), &res.stage1);
    res.st = s;
    if (s != GLOP_OK) res.err = glop_last_error();
    {
      std::lock_guard<std::mutex> lk(gs->res_mu);
      gs->results[w] = std::move(res);
    }
    {
      std::lock_guard<std::mutex> lk(gs->pool_mu);
      gs->pool.push_back(job.second);
    }
    gs->pool_cv.notify_one();
  }
}

uint8_t* gs_take_buffer(glop_group_stream* gs) {
  std::unique_lock<std::mutex> lk(gs->pool_mu);
  gs->pool_cv.wait(lk, [&] { return !gs->pool.empty(); });
  uint8_t* b = gs->pool.back();
  gs->pool.pop_back();
  return b;
}

// hands the filled window (own bytes owned, fill bytes read) to its member
void gs_dispatch(glop_group_stream* gs, uint64_t own) {
  const uint64_t w = gs->windows++;
  {
    std::lock_guard<std::mutex> lk(gs->res_mu);
    gs->results.emplace_back();
    gs->results[w].own = own;
    gs->results[w].read = gs->fill;
  }
  glop_group_stream::Member& mb = *gs->members[w % gs->members.size()];
  {
    std::lock_guard<std::mutex> lk(mb.mu);
    mb.q.emplace_back(w, gs->cur);
  }
  mb.cv.notify_one();
}
}  // namespace

extern "C" {

glop_status glop_group_stream_begin(glop_group* g, const glop_group_trie* t, const glop_group_rules* r,
                                    int with_lines, uint64_t window, glop_group_stream** out) {
  if (!g || !t || !r || !out) return gfail(GLOP_EINVAL, "glop_group_stream_begin: null argument");
  *out = nullptr;
  auto* gs = new glop_group_stream();
  gs->g = g;
  gs->t = t;
  gs->r = r;
  gs->lines = with_lines != 0;
  gs->halo = std::max<uint64_t>(std::max<uint64_t>(t->max_depth, r->max_len), 1) - 1;
  gs->W = std::max<uint64_t>(window ? window : (64ull << 20), gs->halo + 1);
  const size_t nb = 2 * g->ctx.size() + 1;  // two in flight per member + the one being filled
  for (size_t i = 0; i < nb; ++i) {
    void* b = nullptr;
    if (cudaMallocHost(&b, gs->W + gs->halo + 64) != cudaSuccess) {
      cudaGetLastError();
      for (uint8_t* x : gs->all) cudaFreeHost(x);
      delete gs;
      return gfail(GLOP_ENOMEM, "glop_group_stream_begin: pinned window buffers");
    }
    gs->all.push_back(static_cast<uint8_t*>(b));
  }
  gs->pool.assign(gs->all.begin() + 1, gs->all.end());
  gs->cur = gs->all[0];
  for (size_t m = 0; m < g->ctx.size(); ++m) gs->members.push_back(std::make_unique<glop_group_stream::Member>());
  for (size_t m = 0; m < g->ctx.size(); ++m) gs->members[m]->th = std::thread(gs_worker, gs, (int)m);
  *out = gs;
  return GLOP_OK;
}

glop_status glop_group_stream_feed(glop_group_stream* gs, const uint8_t* data, uint64_t len) {
  if (!gs || (len && !data)) return gfail(GLOP_EINVAL, "glop_group_stream_feed: null argument");
  const uint64_t full = gs->W + gs->halo;
  while (len) {
    const uint64_t take = std::min<uint64_t>(len, full - gs->fill);
    parallel_memcpy(gs->cur + gs->fill, data, take);
    gs->fill += take;
    data += take;
    len -= take;
    if (gs->fill == full) {  // window [pos, pos + W) and its halo: hand it over, carry the halo
      uint8_t* next = gs_take_buffer(gs);
      memcpy(next, gs->cur + gs->W, gs->halo);
      gs_dispatch(gs, gs->W);
      gs->cur = next;
      gs->fill = gs->halo;
      gs->pos += gs->W;
    }
  }
  return GLOP_OK;
}

glop_status glop_group_stream_end(glop_group_stream* gs, glop_alert** alerts, uint64_t* n_alerts, uint64_t* counts,
                                  uint64_t* stage1_hits, uint64_t** lines, uint64_t* line_count, uint64_t* bytes) {
  if (!gs) return gfail(GLOP_EINVAL, "glop_group_stream_end: null stream");
  const uint64_t total_bytes = gs->pos + gs->fill;
  if (gs->fill || gs->windows == 0) gs_dispatch(gs, gs->fill);  // the tail owns every remaining start
  for (auto& mb : gs->members) {
    {
      std::lock_guard<std::mutex> lk(mb->mu);
      mb->stop = true;
    }
    mb->cv.notify_one();
  }
  for (auto& mb : gs->members) mb->th.join();
  glop_status s = GLOP_OK;
  std::string err;
  for (auto& res : gs->results)
    if (res.st != GLOP_OK && s == GLOP_OK) s = res.st, err = res.err;
  if (s == GLOP_OK && (!alerts || !n_alerts)) s = GLOP_EINVAL, err = "glop_group_stream_end: null argument";
  if (s == GLOP_OK) {
    std::vector<glop_alert*> pa;
    std::vector<uint64_t> na;
    for (auto& res : gs->results) pa.push_back(res.alerts), na.push_back(res.n_alerts);
    s = concat(pa, na, alerts, n_alerts);
    if (s == GLOP_OK && gs->lines && lines) {
      std::vector<uint64_t*> pl;
      for (auto& res : gs->results) pl.push_back(res.lines);
      uint64_t nl = 0;
      s = concat(pl, na, lines, &nl);
      uint64_t before = 0, at = 0;
      for (size_t w = 0; w < gs->results.size() && s == GLOP_OK; ++w) {
        for (uint64_t i = 0; i < na[w]; ++i) (*lines)[at + i] += before;
        at += na[w];
        before += gs->results[w].line_count - 1;
      }
      if (line_count) *line_count = before + 1;
    }
    if (s == GLOP_OK) {
      if (counts && !gs->results.empty()) {
        const size_t k = gs->results[0].counts.size();
        for (size_t i = 0; i < k; ++i) {
          uint64_t x = 0;
          for (auto& res : gs->results) x += res.counts[i];
          counts[i] = x;
        }
      }
      if (stage1_hits) {
        uint64_t x = 0;
        for (auto& res : gs->results) x += res.stage1;
        *stage1_hits = x;
      }
      if (bytes) *bytes = total_bytes;
    }
  } else {
    gfail(s, err);
  }
  for (auto& res : gs->results) {
    glop_free(res.alerts);
    glop_free(res.lines);
  }
  for (uint8_t* b : gs->all) cudaFreeHost(b);
  delete gs;
  return s;
}

}  // extern "C"
