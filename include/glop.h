/*
 * glop.h -- C ABI of the B200-native GLoP matching path (libglop.so).
 *
 * This is the drop-in boundary underneath the reference's C++ API
 * (namespace logtrawl, /root/reference/proj/include/logtrawl/*.hpp).  The C++
 * headers in include/logtrawl/ keep the reference signatures and call these
 * entry points; every entry point below names the reference interface it
 * replaces.  Plain pointers and sizes only; no torch or C++ types.
 *
 * Conventions
 *  - Every function returns a glop_status; on failure glop_last_error()
 *    returns a thread-local message.  The C++ shim maps codes onto the
 *    reference's exception types (see include/logtrawl/detail/abi.hpp).
 *  - "host" pointers may be pageable or pinned; "device" pointers are CUDA
 *    device pointers on the context's device.
 *  - Arrays returned through `T** out` are library-owned host memory, released
 *    with glop_free().
 *  - A glop_ctx owns one CUDA stream plus scratch; calls on one context are
 *    serialised, calls on different contexts run concurrently.  A glop_trie /
 *    glop_rules is immutable after upload and may be shared by contexts on the
 *    same device (automaton.hpp "immutable value, shareable").
 *  - There is no CPU fallback: without a usable sm_100 device, calls fail with
 *    GLOP_ECUDA.
 */
#ifndef GLOP_H_
#define GLOP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GLOP_OK = 0,
  GLOP_EINVAL = 1,    /* reference: std::invalid_argument              */
  GLOP_ECAPACITY = 2, /* reference: logtrawl::CapacityError            */
  GLOP_ELOGIC = 3,    /* reference: std::logic_error (verify.hpp:76-77) */
  GLOP_ECUDA = 4,     /* device / driver failure (std::runtime_error)   */
  GLOP_ENOMEM = 5,    /* allocation failure (std::bad_alloc)            */
  GLOP_EAGAIN = 6     /* an asynchronous call must be redone synchronously */
} glop_status;

/* Layout-identical to logtrawl::Hit (scan.hpp:31-41) on LP64: 16 bytes. */
typedef struct {
  uint64_t offset;
  uint32_t pattern_id;
  uint32_t matched_len;
} glop_hit;

/* Layout-identical to logtrawl::AutomatonOutput (automaton.hpp:43-49). */
typedef struct {
  uint32_t pattern_id;
  uint32_t matched_len;
} glop_output;

/* Verified match (verify.hpp:19-28 Alert without the name string / line). */
typedef struct {
  uint64_t offset;
  uint32_t rule_id;
  uint32_t pattern_len;
} glop_alert;

typedef struct glop_ctx glop_ctx;
typedef struct glop_trie glop_trie;
typedef struct glop_rules glop_rules;

/* PFAC kernel selection.  FILTERED is the general q-gram-filtered kernel
 * (the GPU analogue of the reference's RootJump, scan.hpp:81-108); PREFIX8
 * the lean kernel for automata whose outputs all lie at depth >= 8 (8-byte
 * prefixes: aligned 4-gram sampling + 8-byte key bitmap); DIRECT the literal
 * one-thread-per-byte walk (scan.hpp:113-170).  AUTO picks PREFIX8 when it
 * applies, else FILTERED.  All are exact and return identical results. */
typedef enum {
  GLOP_PFAC_AUTO = 0,
  GLOP_PFAC_FILTERED = 1,
  GLOP_PFAC_DIRECT = 2,
  GLOP_PFAC_PREFIX8 = 3
} glop_pfac_kernel;

const char* glop_last_error(void);
const char* glop_version(void);

/* ---- context ------------------------------------------------------------ */
glop_status glop_ctx_create(int device, glop_ctx** out);
glop_status glop_ctx_destroy(glop_ctx* ctx);
/* The context's CUDA stream (cudaStream_t as void*), for callers that want to
 * order their own work (events, NCCL) against library calls. */
void* glop_ctx_stream(glop_ctx* ctx);
glop_status glop_ctx_synchronize(glop_ctx* ctx);

/* ---- automaton ------------------------------------------------------------
 * Replaces the consumer side of build_failureless_trie (automaton.hpp:283-291):
 * takes the reference's own dense representation -- Q x 256 int32 goto table
 * with -1 = no edge (automaton.hpp:57), CSR outputs out_offsets[Q+1] /
 * out_flat (automaton.hpp:78-79) -- and flattens it once into the device
 * layout: byte->class map, alphabet-compressed transition table (u16 entries
 * when Q < 32768), per-pattern lengths and the q-gram filter tables.
 * Fails with GLOP_EINVAL if the input is not a failureless trie (an edge to
 * the root, a state with two parents, an unreachable state). */
glop_status glop_trie_upload(glop_ctx* ctx, const int32_t* dense_table, uint32_t state_count,
                             const uint32_t* out_offsets, const glop_output* out_flat,
                             glop_trie** out);
glop_status glop_trie_destroy(glop_trie* trie);
/* Introspection for tests: state count, alphabet classes, min/max output
 * depth, filter q-gram length and stride, table bytes, whether the table is
 * staged in shared memory by the filtered kernel, the jump-table depth J and
 * slot count and whether it is staged in shared memory. */
typedef struct {
  uint32_t state_count, classes, min_depth, max_depth, q, stride, entry_bytes, table_in_smem;
  uint64_t table_bytes;
  uint32_t jump_depth, jump_in_smem, jump_slots, reserved;
} glop_trie_info;
glop_status glop_trie_get_info(const glop_trie* trie, glop_trie_info* info);

/* ---- PFAC scan ------------------------------------------------------------
 * Replaces pfac_scan (scan.hpp:177-202): every start position of `text`
 * walks the failureless trie; a Hit is emitted for every output of every
 * visited state; the result is sorted by (offset, pattern_id).
 * glop_pfac_scan: host-facing; `text_on_device` says where text lives; the
 * result is a library-owned host array (glop_free). */
glop_status glop_pfac_scan(glop_ctx* ctx, const glop_trie* trie, const uint8_t* text, uint64_t n,
                           int text_on_device, glop_hit** hits, uint64_t* n_hits);

/* Shard form: text covers global offsets [base, base+n); only starts in
 * [base, base+own) are reported (the bytes past own are the halo). */
glop_status glop_pfac_scan_shard(glop_ctx* ctx, const glop_trie* trie, const uint8_t* text, uint64_t n,
                                 uint64_t own, uint64_t base, int text_on_device, glop_hit** hits,
                                 uint64_t* n_hits);

/* Device-resident form for shards and pipelines: reads text[0, n) (device),
 * reports only starts in [0, own) (own <= n; the bytes [own, n) are the halo),
 * adds `base` to every reported offset, and writes the sorted hits to
 * out[0, min(cap, total)).  *n_hits is the total; if it exceeds cap the call
 * returns GLOP_ECAPACITY and the caller retries with a larger buffer. */
glop_status glop_pfac_scan_device(glop_ctx* ctx, const glop_trie* trie, const uint8_t* d_text,
                                  uint64_t n, uint64_t own, uint64_t base, glop_pfac_kernel kernel,
                                  glop_hit* d_out, uint64_t cap, uint64_t* n_hits);

/* ---- streaming ingest ----------------------------------
 * run_engine_scan's PFAC branch over a text that arrives in pieces (a file
 * read in windows, a log tail): the result equals glop_run_pfac_pipeline[_lines]
 * over the concatenation of every fed piece.  Windows of 256 MiB are scanned
 * as they fill; each reads max(trie depth, longest pattern) - 1 bytes of the
 * next, carried across feed() calls (SPEC.md:290's max_len-1 windowing), so a
 * match straddling two pieces is reported once, by the window owning its
 * start.  glop_stream_end returns the results (library-owned arrays, as
 * glop_run_pfac_pipeline_lines; lines/line_count may be NULL when the stream
 * was begun without lines; bytes = total fed) and frees the stream, also on
 * error.  One stream at a time per context is not required: feeds lock the
 * context only while a window is scanned. */
typedef struct glop_stream glop_stream;
glop_status glop_stream_begin(glop_ctx* ctx, const glop_trie* trie, const glop_rules* rules, int with_lines,
                              glop_stream** out);
glop_status glop_stream_feed(glop_stream* stream, const uint8_t* data, uint64_t len);
glop_status glop_stream_end(glop_stream* stream, glop_alert** alerts, uint64_t* n_alerts, uint64_t* counts,
                            uint64_t* stage1_hits, uint64_t** lines, uint64_t* line_count, uint64_t* bytes);

/* ---- chunked full Aho-Corasick --------------------------------------------
 * Replaces chunked_ac_scan (scan.hpp:207-243): chunk k owns starts
 * [k*c, (k+1)*c) (c = chunk_size, 0 = the whole text) and is scanned from the
 * root over [k*c, min(k*c + c + overlap, n)); a match is reported iff the
 * chunk owning its start also reaches its end -- so an overlap below
 * max_len - 1 loses boundary-straddling matches exactly as the reference does.
 * `trie` is the GOTO trie of the AC automaton (its dense table) with only each
 * pattern's own output (matched_len == depth); the device enumerates every
 * occurrence with the PFAC kernel and keeps the owned, reached ones.  Result:
 * (offset, pattern_id, matched_len) records sorted by (offset, pattern_id),
 * library-owned (glop_free). */
glop_status glop_chunked_ac_scan(glop_ctx* ctx, const glop_trie* trie, const uint8_t* text, uint64_t n,
                                 int text_on_device, uint64_t chunk_size, uint64_t overlap, glop_hit** matches,
                                 uint64_t* n_matches);

/* ---- end-to-end PFAC pipeline --------------------------------------------
 * The device half of run_engine_scan's PFAC branch (pipeline.hpp:86-97):
 * text (host or device) -> pfac_scan -> verify_hits -> alerts + per-pattern
 * counts, one host->device copy of the text and one device->host copy of the
 * alerts.  `counts` (optional, host, n_patterns u64) receives the alert
 * histogram; `stage1_hits` the pre-verification hit count. */
glop_status glop_run_pfac_pipeline(glop_ctx* ctx, const glop_trie* trie, const glop_rules* rules,
                                   const uint8_t* text, uint64_t n, int text_on_device,
                                   glop_alert** alerts, uint64_t* n_alerts, uint64_t* counts,
                                   uint64_t* stage1_hits);
/* Shard form: text covers global offsets [base, base+n); only starts in
 * [base, base+own) are reported. */
glop_status glop_run_pfac_pipeline_shard(glop_ctx* ctx, const glop_trie* trie,
                                         const glop_rules* rules, const uint8_t* text, uint64_t n,
                                         uint64_t own, uint64_t base, int text_on_device,
                                         glop_alert** alerts, uint64_t* n_alerts, uint64_t* counts,
                                         uint64_t* stage1_hits);

/* With a LineIndex (run_engine_scan's `lines` argument, pipeline.hpp:49 /
 * verify.hpp:40-64): also lines[i] = LineIndex(text).line_of(alerts[i].offset)
 * (library-owned, glop_free) and *line_count = LineIndex(text).line_count()
 * (1 + LF bytes of text), computed on the device from the same upload. */
glop_status glop_run_pfac_pipeline_lines(glop_ctx* ctx, const glop_trie* trie, const glop_rules* rules,
                                         const uint8_t* text, uint64_t n, int text_on_device, glop_alert** alerts,
                                         uint64_t* n_alerts, uint64_t* counts, uint64_t* stage1_hits,
                                         uint64_t** lines, uint64_t* line_count);

/* Shard form of the above: lines[i] counts lines within the shard's owned
 * bytes [0, own) (1 + LFs of text[0, alerts[i].offset - base)) and
 * *line_count = 1 + LF bytes in text[0, own); a caller adds the LFs of the
 * shards before this one (glop_group_run_pfac_pipeline does). */
glop_status glop_run_pfac_pipeline_shard_lines(glop_ctx* ctx, const glop_trie* trie, const glop_rules* rules,
                                               const uint8_t* text, uint64_t n, uint64_t own, uint64_t base,
                                               int text_on_device, glop_alert** alerts, uint64_t* n_alerts,
                                               uint64_t* counts, uint64_t* stage1_hits, uint64_t** lines,
                                               uint64_t* line_count);

/* Fully device-resident form (the bench step): d_text holds global offsets
 * [base, base+n); starts [base, base+own) are scanned.  Writes the sorted
 * alerts to d_alerts[0, alert_cap), the per-pattern alert counts to d_counts
 * (n_patterns u64, OVERWRITTEN; may be NULL) and, when d_hits is not NULL,
 * the sorted stage-1 hits to d_hits[0, hit_cap).  For 8-byte-prefix automata
 * every kernel is enqueued back to back and the host waits once, at the end.
 * GLOP_ECAPACITY (with *n_hits / *n_alerts set to the totals) when a buffer
 * is too small. */
glop_status glop_run_pfac_pipeline_device(glop_ctx* ctx, const glop_trie* trie, const glop_rules* rules,
                                          const uint8_t* d_text, uint64_t n, uint64_t own, uint64_t base,
                                          glop_hit* d_hits, uint64_t hit_cap, glop_alert* d_alerts,
                                          uint64_t alert_cap, uint64_t* d_counts, uint64_t* n_hits,
                                          uint64_t* n_alerts);

/* Asynchronous form for pipelined submission (a stream of shards, the bench
 * step): enqueues the same work and returns without waiting; the status block
 * is copied (stream-ordered) into *ticket, which must stay valid -- pinned
 * host memory (glop_host_alloc) -- until the context stream is synchronized.
 * Then glop_pipeline_ticket_result gives (n_hits, n_alerts) or the error; it
 * returns GLOP_EAGAIN when this input needs the synchronous call (a hit-dense
 * input that overflowed a warp's hit buffer or staging region: its outputs are
 * not valid, rerun it with glop_run_pfac_pipeline_device).  Automata without
 * the fused path run synchronously here and complete the ticket at once. */
typedef struct {
  uint64_t raw[8];  /* device status block */
  uint64_t region, hit_cap, alert_cap;
  uint32_t stage2, done;
} glop_pipeline_ticket;
glop_status glop_run_pfac_pipeline_device_async(glop_ctx* ctx, const glop_trie* trie, const glop_rules* rules,
                                                const uint8_t* d_text, uint64_t n, uint64_t own, uint64_t base,
                                                glop_hit* d_hits, uint64_t hit_cap, glop_alert* d_alerts,
                                                uint64_t alert_cap, uint64_t* d_counts,
                                                glop_pipeline_ticket* ticket);
glop_status glop_pipeline_ticket_result(const glop_pipeline_ticket* ticket, uint64_t* n_hits, uint64_t* n_alerts);

/* ---- measurement ----------------------------------------------------------
 * Device time of the most recent PFAC / KMP scan kernel on this context,
 * from CUDA events recorded on the context stream around the launch. */
glop_status glop_last_kernel_ms(glop_ctx* ctx, float* ms);
/* Number of kernels this context has launched so far. */
uint64_t glop_ctx_launch_count(glop_ctx* ctx);
/* Number of PFAC scans on this context that needed the exact global-key
 * fallback (one lane emitting more hits than a warp's hit buffer holds). */
uint64_t glop_ctx_fallback_count(glop_ctx* ctx);

/* ---- stage-2 verification ------------------------------------------------
 * Patterns for verify_hits (verify.hpp:69-105): bytes of pattern i are
 * bytes[off[i], off[i+1]), its id is i (rules.hpp:24-33). */
glop_status glop_rules_upload(glop_ctx* ctx, const uint8_t* bytes, const uint64_t* off,
                              uint32_t n_patterns, uint64_t prefix_len, glop_rules** out);
glop_status glop_rules_destroy(glop_rules* rules);

/* verify_hits: keeps hits whose pattern suffix matches (patterns no longer
 * than prefix_len are auto-verified; a pattern running past the end of text
 * is rejected); alerts sorted by (offset, rule_id).  GLOP_ELOGIC if a hit
 * extends past the end of text or names an unknown pattern (verify.hpp:76-77,
 * rules.patterns.at()).  Host-facing; alerts are a library-owned host array.
 * `counts` (optional, host, n_patterns entries) receives the per-pattern
 * alert histogram. */
glop_status glop_verify_hits(glop_ctx* ctx, const glop_rules* rules, const uint8_t* text,
                             uint64_t n, int text_on_device, const glop_hit* hits, uint64_t n_hits,
                             int hits_on_device, glop_alert** alerts, uint64_t* n_alerts,
                             uint64_t* counts);

/* Device-resident verify: hits/text/out/counts are device pointers; d_text
 * holds global offsets [base, base+n) (base = 0 for a whole text; a shard's
 * first owned offset otherwise -- hits carry global offsets).  counts
 * (n_patterns u64, may be NULL) is ACCUMULATED into.  out must hold n_hits. */
glop_status glop_verify_hits_device(glop_ctx* ctx, const glop_rules* rules, const uint8_t* d_text,
                                    uint64_t n, uint64_t base, const glop_hit* d_hits,
                                    uint64_t n_hits, glop_alert* d_out, uint64_t* n_alerts,
                                    uint64_t* d_counts);

/* ---- LineIndex ------------------------------------------------------------
 * Replaces LineIndex(text).line_of(offset) (verify.hpp:40-64) for many
 * offsets at once: line = 1 + number of LF bytes before the offset (an LF
 * belongs to the line it ends).  One HBM pass counts LFs per 4 KB block, a
 * device scan makes them prefixes, one warp per offset finishes the count.
 * glop_line_numbers: host offsets/lines (offsets <= n, else GLOP_EINVAL).
 * glop_line_numbers_device: records are `stride`-byte structs whose first 8
 * bytes are a global offset in [base, base+n) (glop_hit / glop_alert: stride
 * 16; plain u64: 8); d_text holds global offsets [base, base+n). */
glop_status glop_line_numbers(glop_ctx* ctx, const uint8_t* text, uint64_t n, int text_on_device,
                              const uint64_t* offsets, uint64_t count, uint64_t* lines);
glop_status glop_line_numbers_device(glop_ctx* ctx, const uint8_t* d_text, uint64_t n, uint64_t base,
                                     const void* d_records, uint32_t stride, uint64_t count,
                                     uint64_t* d_lines);

/* ---- KMP ------------------------------------------------------------------
 * Replaces kmp_search (kmp.hpp:41-69): all start offsets (ascending,
 * overlapping included) of pattern p; `failure` is the reference failure
 * table (kmp.hpp:25-36), m entries.  `comparisons` (optional) is incremented
 * by exactly the number of byte comparisons the sequential algorithm makes.
 * Runs chunk-parallel with an (m-1)-byte warm-up overlap per chunk. */
glop_status glop_kmp_search(glop_ctx* ctx, const uint8_t* p, uint32_t m, const uint32_t* failure,
                            const uint8_t* text, uint64_t n, int text_on_device, uint64_t** offsets,
                            uint64_t* n_offsets, uint64_t* comparisons);
/* Host-facing shard form: text = global offsets [base, base+n); starts at
 * local positions [skip, own) are reported (as base + start) and the
 * comparisons the sequential scan makes at positions [skip, own) are added.
 * Exact when skip = 0 is the true text start or skip >= m - 1 (a left context
 * from which the KMP state is recovered); shards [lo_g, hi_g) read with
 * min(lo_g, m-1) bytes of left context and m-1 bytes of right halo sum to the
 * whole-text result, comparisons included. */
glop_status glop_kmp_search_shard(glop_ctx* ctx, const uint8_t* p, uint32_t m, const uint32_t* failure,
                                  const uint8_t* text, uint64_t n, uint64_t skip, uint64_t own, uint64_t base,
                                  int text_on_device, uint64_t** offsets, uint64_t* n_offsets,
                                  uint64_t* comparisons);
/* Shard form: d_text holds global offsets [base, base+n); reports the
 * starts in [0, own) (matches may end in the halo [own, own+m-1)), adds
 * `base` to each, and counts the comparisons the sequential scan makes at
 * positions [0, own) -- so shards with an (m-1)-byte halo sum to the whole. */
glop_status glop_kmp_search_device(glop_ctx* ctx, const uint8_t* p, uint32_t m,
                                   const uint32_t* failure, const uint8_t* d_text, uint64_t n,
                                   uint64_t own, uint64_t base, uint64_t* d_out, uint64_t cap,
                                   uint64_t* n_offsets, uint64_t* comparisons);

/* ---- multi-GPU group ------------------------------------------
 * One context per member device; `devices` may repeat a device (N contexts on
 * one GPU exercise the N-way split on a one-GPU box); devices == NULL takes
 * the first n_devices visible devices (n_devices <= 0: all of them).  A group
 * call splits the text into contiguous shards (member g owns starts
 * [lo_g, lo_g + own_g) and reads a halo of max(trie depth, longest pattern)
 * - 1 bytes past them -- scan.hpp:59-79 ranges, scan.hpp:230-232 ownership),
 * runs each shard on its member's stream from its own host thread, and merges
 * in rank order: results are byte-identical to one context's.  Shards are at
 * least GLOP_GROUP_MIN_SHARD bytes (default 64 MiB), so small texts use fewer
 * members.  Host text only (pageable or pinned); results are library-owned
 * host arrays (glop_free). */
typedef struct glop_group glop_group;
typedef struct glop_group_trie glop_group_trie;
typedef struct glop_group_rules glop_group_rules;
glop_status glop_group_create(const int* devices, int n_devices, glop_group** out);
glop_status glop_group_destroy(glop_group* group);
int glop_group_size(const glop_group* group);
glop_ctx* glop_group_ctx(glop_group* group, int member);
glop_status glop_group_trie_upload(glop_group* group, const int32_t* dense_table, uint32_t state_count,
                                   const uint32_t* out_offsets, const glop_output* out_flat, glop_group_trie** out);
glop_trie* glop_group_trie_member(glop_group_trie* trie, int member);
glop_status glop_group_trie_destroy(glop_group_trie* trie);
glop_status glop_group_rules_upload(glop_group* group, const uint8_t* bytes, const uint64_t* off, uint32_t n_patterns,
                                    uint64_t prefix_len, glop_group_rules** out);
glop_rules* glop_group_rules_member(glop_group_rules* rules, int member);
glop_status glop_group_rules_destroy(glop_group_rules* rules);
/* pfac_scan (scan.hpp:177-202) over all members. */
glop_status glop_group_pfac_scan(glop_group* group, const glop_group_trie* trie, const uint8_t* text, uint64_t n,
                                 glop_hit** hits, uint64_t* n_hits);
/* run_engine_scan's PFAC branch over all members: alerts, counts (optional,
 * n_patterns u64), stage-1 hits, and (lines and line_count both given, or
 * both NULL) LineIndex(text) line numbers / line count. */
glop_status glop_group_run_pfac_pipeline(glop_group* group, const glop_group_trie* trie, const glop_group_rules* rules,
                                         const uint8_t* text, uint64_t n, glop_alert** alerts, uint64_t* n_alerts,
                                         uint64_t* counts, uint64_t* stage1_hits, uint64_t** lines,
                                         uint64_t* line_count);
/* kmp_search (kmp.hpp:41-69) over all members; comparisons exact (each shard
 * reads m-1 bytes of left context to recover the KMP state). */
glop_status glop_group_kmp_search(glop_group* group, const uint8_t* p, uint32_t m, const uint32_t* failure,
                                  const uint8_t* text, uint64_t n, uint64_t** offsets, uint64_t* n_offsets,
                                  uint64_t* comparisons);
/* Streaming over the group: windows of `window` bytes (0 = 64 MiB) -- each
 * reading the next window's first max(depth, max_len) - 1 bytes, carried
 * across feed() calls -- go round-robin to the members, which scan them
 * concurrently (one host thread, stream and PCIe link each); end() merges in
 * window order: the results equal glop_run_pfac_pipeline[_lines] over the
 * concatenation (lines / line_count as in glop_stream_end). */
typedef struct glop_group_stream glop_group_stream;
glop_status glop_group_stream_begin(glop_group* group, const glop_group_trie* trie, const glop_group_rules* rules,
                                    int with_lines, uint64_t window, glop_group_stream** out);
glop_status glop_group_stream_feed(glop_group_stream* stream, const uint8_t* data, uint64_t len);
glop_status glop_group_stream_end(glop_group_stream* stream, glop_alert** alerts, uint64_t* n_alerts,
                                  uint64_t* counts, uint64_t* stage1_hits, uint64_t** lines, uint64_t* line_count,
                                  uint64_t* bytes);
/* The shard plan (host only, no device): parts contiguous ranges, the first
 * n % parts one byte longer; read = min(own + halo, n - lo). */
glop_status glop_plan_shards(uint64_t n, uint32_t parts, uint64_t halo, uint64_t* lo, uint64_t* own,
                             uint64_t* read);

/* Asynchronous device KMP (pipelined submission, as
 * glop_run_pfac_pipeline_device_async): the status lands in *ticket (pinned);
 * after the context stream is synchronized glop_kmp_ticket_result gives the
 * number of offsets and ADDS the comparisons, or GLOP_EAGAIN when the input
 * needs the synchronous call (a match-dense tile or a staging overflow). */
glop_status glop_kmp_search_device_async(glop_ctx* ctx, const uint8_t* p, uint32_t m, const uint32_t* failure,
                                         const uint8_t* d_text, uint64_t n, uint64_t own, uint64_t base,
                                         uint64_t* d_out, uint64_t cap, glop_pipeline_ticket* ticket);
glop_status glop_kmp_ticket_result(const glop_pipeline_ticket* ticket, uint64_t* n_offsets, uint64_t* comparisons);

/* ---- memory helpers -------------------------------------------------------- */
void glop_free(void* p);
glop_status glop_device_alloc(glop_ctx* ctx, uint64_t bytes, void** out);
glop_status glop_device_free(glop_ctx* ctx, void* p);
glop_status glop_host_alloc(uint64_t bytes, void** out); /* pinned */
glop_status glop_host_free(void* p);
glop_status glop_memcpy(glop_ctx* ctx, void* dst, const void* src, uint64_t bytes, int kind);
/* kind: 1 = host->device, 2 = device->host, 3 = device->device (stream-ordered) */

/* ---- host-side automaton construction (drop-in C++ code, exported for
 * FFI callers such as the Python test/bench harness) ------------------------
 * truncate_prefixes (rules.hpp:190-208) + build_failureless_trie
 * (automaton.hpp:283-291) exactly as include/logtrawl/ implements them; the
 * result is the reference's dense form, ready for glop_trie_upload.  Arrays
 * are library-owned (glop_free).  GLOP_EINVAL for prefix_len < 1,
 * GLOP_ECAPACITY when the trie would exceed max_states. */
glop_status glop_build_failureless_trie(const uint8_t* bytes, const uint64_t* off, uint32_t n_patterns,
                                        uint64_t prefix_len, uint64_t max_states, int32_t** dense_table,
                                        uint32_t* state_count, uint32_t** out_offsets,
                                        glop_output** out_flat);

/* ---- synthetic workloads (bench / tests; not the matching path) ------------ */
/* Bytes [begin, begin+n) of synthetic RFC 5424 corpus `seed`
 * (paper_1704_02278_b200/csrc/corpus.h); device and host forms are
 * byte-identical. */
glop_status glop_gen_syslog_device(glop_ctx* ctx, uint8_t* d_out, uint64_t begin, uint64_t n,
                                   uint64_t seed);
glop_status glop_gen_syslog_host(uint8_t* out, uint64_t begin, uint64_t n, uint64_t seed,
                                 unsigned threads);
/* Bytes [begin, begin+n) of synthetic packet-payload stream `seed` (DPI
 * configuration, paper_1704_02278_b200/csrc/payload.h); device and host forms
 * are byte-identical. */
glop_status glop_gen_payload_device(glop_ctx* ctx, uint8_t* d_out, uint64_t begin, uint64_t n,
                                    uint64_t seed);
glop_status glop_gen_payload_host(uint8_t* out, uint64_t begin, uint64_t n, uint64_t seed,
                                  unsigned threads);
/* Snort-style content rules for the DPI configuration: k distinct contents of
 * min_len..max_len bytes (half random full-byte, half payload windows).
 * bytes must hold k*max_len; off receives k+1 offsets. */
glop_status glop_gen_dpi_rules(uint32_t k, uint32_t seed, uint32_t min_len, uint32_t max_len,
                               uint8_t* bytes, uint64_t* off);
/* Reference corpus semantics (loggen.hpp:44-57), host only. */
glop_status glop_gen_reference_log(uint8_t* out, uint64_t size, uint32_t seed, uint64_t line_len);
/* Synthetic rule set: k patterns of `len` bytes, half with the reference's
 * random_rules semantics (loggen.hpp:60-78), half sampled from the corpus's
 * incident vocabulary.  bytes must hold k*len; names are "rand-i"/"vocab-i"
 * (is_vocab[i] = 1 for vocabulary patterns; may be NULL). */
glop_status glop_gen_rules(uint32_t k, uint32_t seed, uint32_t len, uint8_t* bytes,
                           uint8_t* is_vocab);

/* ---- peer exchange between processes (one process per GPU) --------------
 * The one exchange of the sharded path (per-rank alert lists
 * to the root, per-pattern counts) done with CUDA IPC and copy-engine
 * copies over NVLink instead of NCCL kernels: a persistent scan kernel holds
 * every SM, so an SM-based collective on another stream could not start
 * until it ends, while copy engines run beside it.  Handles are 64 opaque
 * bytes the caller moves between processes (e.g. torch.distributed object
 * collectives); streams are cudaStream_t as void* (glop_ctx_stream).
 *   glop_peer_alloc       device buffer on ctx's device + its IPC handle
 *   glop_peer_open        map another process's buffer (any device)
 *   glop_peer_event       interprocess event + its handle;
 *   glop_peer_event_open  the other process's event
 *   glop_peer_record / glop_peer_wait   event record on / wait by a stream
 *   glop_peer_copy        async device-to-device copy on a stream (copy engine) */
glop_status glop_peer_alloc(glop_ctx* ctx, uint64_t bytes, void** d_ptr, void* handle64);
glop_status glop_peer_free(glop_ctx* ctx, void* d_ptr);
glop_status glop_peer_open(glop_ctx* ctx, const void* handle64, void** d_ptr);
glop_status glop_peer_close(glop_ctx* ctx, void* d_ptr);
glop_status glop_peer_event(glop_ctx* ctx, void** event, void* handle64);
glop_status glop_peer_event_open(glop_ctx* ctx, const void* handle64, void** event);
glop_status glop_peer_event_destroy(glop_ctx* ctx, void* event);
glop_status glop_peer_record(glop_ctx* ctx, void* event, void* stream);
glop_status glop_peer_wait(glop_ctx* ctx, void* stream, void* event);
glop_status glop_peer_copy(glop_ctx* ctx, void* dst, const void* src, uint64_t bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GLOP_H_ */
