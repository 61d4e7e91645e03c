/*
 * pfac_oracle.c -- CPU restatement of the logtrawl matching path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * kernels: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it.  The product path (libglop.so) never links or calls it.
 *
 * Parity is PINNED: tests/test_oracle.py checks every function here against
 * golden vectors produced by the unmodified reference (oracle/gen_golden.cpp
 * compiled against /root/reference/proj/include, fixtures under
 * tests/golden/) and against the reference's own known-answer tests.
 *
 * Each function cites the reference code it restates (paths relative to
 * /root/reference/proj/include/logtrawl/).  Plain C99, single-threaded,
 * written for clarity, not speed.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL 1    /* std::invalid_argument */
#define OR_ECAPACITY 2 /* CapacityError        */
#define OR_ELOGIC 3    /* std::logic_error     */
#define OR_ENOMEM 5

typedef struct {
  uint64_t offset;
  uint32_t pattern_id;
  uint32_t matched_len;
} or_hit; /* scan.hpp:31-41 (Hit) */

typedef struct {
  uint32_t pattern_id;
  uint32_t matched_len;
} or_output; /* automaton.hpp:43-49 (AutomatonOutput) */

typedef struct {
  uint64_t offset;
  uint32_t rule_id;
  uint32_t pattern_len;
  uint64_t line;
} or_alert; /* verify.hpp:19-28 (Alert), name dropped */

/* A pattern set is passed as concatenated bytes + (n+1) offsets; pattern i
 * is bytes[off[i] .. off[i+1]) and has id i (rules.hpp:24-33). */

/* ---------------------------------------------------------------------- */
/* truncate_prefixes (rules.hpp:190-208)                                   */
/* entries: first-appearance order; entry_of[pid] = entry index.           */
/* Returns number of entries; entry_src[e] = first pattern id of entry e.  */
/* ---------------------------------------------------------------------- */
int or_truncate_prefixes(const uint8_t* bytes, const uint64_t* off,
                         uint32_t n_patterns, uint64_t prefix_len,
                         uint32_t* entry_of, uint32_t* entry_src,
                         uint32_t* entry_len, uint32_t* n_entries) {
  if (prefix_len < 1) return OR_EINVAL; /* rules.hpp:192-193 */
  uint32_t ne = 0;
  for (uint32_t p = 0; p < n_patterns; ++p) {
    uint64_t len = off[p + 1] - off[p];
    uint64_t pl = len < prefix_len ? len : prefix_len;
    uint32_t hit = UINT32_MAX;
    /* quadratic lookup is fine for an oracle (map in rules.hpp:196) */
    for (uint32_t e = 0; e < ne && hit == UINT32_MAX; ++e) {
      if (entry_len[e] == pl &&
          memcmp(bytes + off[entry_src[e]], bytes + off[p], pl) == 0)
        hit = e;
    }
    if (hit == UINT32_MAX) {
      entry_src[ne] = p;
      entry_len[ne] = (uint32_t)pl;
      hit = ne++;
    }
    entry_of[p] = hit;
  }
  *n_entries = ne;
  return OR_OK;
}

/* ---------------------------------------------------------------------- */
/* build_failureless_trie (automaton.hpp:147-212, 283-291)                 */
/* Insertion trie with 256-wide child rows, then BFS renumbering with      */
/* children visited in ascending byte order.  Outputs of the node where    */
/* entry e ends = all ids of e in id order, matched_len = |prefix|.        */
/* ---------------------------------------------------------------------- */
typedef struct {
  uint32_t state_count;
  int32_t* table;        /* state_count * 256, -1 = no edge */
  uint32_t* depth;       /* state_count */
  uint32_t* out_offsets; /* state_count + 1 */
  or_output* out_flat;
  uint32_t n_out;
} or_trie;

void or_trie_free(or_trie* t) {
  if (!t) return;
  free(t->table);
  free(t->depth);
  free(t->out_offsets);
  free(t->out_flat);
  free(t);
}

int or_build_trie(const uint8_t* bytes, const uint64_t* off,
                  uint32_t n_patterns, uint64_t prefix_len,
                  uint64_t max_states, or_trie** out) {
  *out = NULL;
  if (prefix_len < 1) return OR_EINVAL;
  uint32_t* entry_of = malloc(sizeof(uint32_t) * (n_patterns + 1));
  uint32_t* entry_src = malloc(sizeof(uint32_t) * (n_patterns + 1));
  uint32_t* entry_len = malloc(sizeof(uint32_t) * (n_patterns + 1));
  uint32_t ne = 0;
  or_truncate_prefixes(bytes, off, n_patterns, prefix_len, entry_of,
                       entry_src, entry_len, &ne);

  /* insertion trie: children rows, node -> entry that ends there */
  uint64_t cap = 1 + 16;
  int32_t* rows = malloc(sizeof(int32_t) * 256 * cap);
  int32_t* ends = malloc(sizeof(int32_t) * cap);
  memset(rows, 0xff, sizeof(int32_t) * 256);
  ends[0] = -1;
  uint64_t nn = 1;
  int rc = OR_OK;
  for (uint32_t e = 0; e < ne && rc == OR_OK; ++e) {
    const uint8_t* s = bytes + off[entry_src[e]];
    int32_t cur = 0;
    for (uint32_t k = 0; k < entry_len[e]; ++k) {
      int32_t nx = rows[(uint64_t)cur * 256 + s[k]];
      if (nx < 0) {
        if (nn >= max_states) { /* automaton.hpp:163 */
          rc = OR_ECAPACITY;
          break;
        }
        if (nn == cap) {
          cap *= 2;
          rows = realloc(rows, sizeof(int32_t) * 256 * cap);
          ends = realloc(ends, sizeof(int32_t) * cap);
        }
        memset(rows + nn * 256, 0xff, sizeof(int32_t) * 256);
        ends[nn] = -1;
        nx = (int32_t)nn++;
        rows[(uint64_t)cur * 256 + s[k]] = nx;
      }
      cur = nx;
    }
    if (rc == OR_OK) ends[cur] = (int32_t)e;
  }
  if (rc != OR_OK) {
    free(rows), free(ends), free(entry_of), free(entry_src), free(entry_len);
    return rc;
  }

  /* BFS renumbering (automaton.hpp:198-212) */
  int32_t* order = malloc(sizeof(int32_t) * nn);   /* new -> old */
  int32_t* renum = malloc(sizeof(int32_t) * nn);   /* old -> new */
  uint64_t head = 0, tail = 0;
  order[tail++] = 0;
  renum[0] = 0;
  while (head < tail) {
    int32_t old = order[head++];
    for (int b = 0; b < 256; ++b) {
      int32_t c = rows[(uint64_t)old * 256 + b];
      if (c >= 0) {
        renum[c] = (int32_t)tail;
        order[tail++] = c;
      }
    }
  }
  or_trie* t = calloc(1, sizeof(or_trie));
  t->state_count = (uint32_t)nn;
  t->table = malloc(sizeof(int32_t) * 256 * nn);
  t->depth = calloc(nn, sizeof(uint32_t));
  t->out_offsets = malloc(sizeof(uint32_t) * (nn + 1));
  t->out_flat = malloc(sizeof(or_output) * (n_patterns + 1));
  uint32_t no = 0;
  for (uint64_t ns = 0; ns < nn; ++ns) {
    int32_t old = order[ns];
    for (int b = 0; b < 256; ++b) {
      int32_t c = rows[(uint64_t)old * 256 + b];
      int32_t nc = c >= 0 ? renum[c] : -1;
      t->table[ns * 256 + b] = nc;
      if (nc >= 0) t->depth[nc] = t->depth[ns] + 1;
    }
    /* CSR outputs (automaton.hpp:132-140): all ids of the entry ending
     * here, in the entry's id order (rules.hpp:200-205). */
    t->out_offsets[ns] = no;
    if (ends[old] >= 0) {
      uint32_t e = (uint32_t)ends[old];
      for (uint32_t p = 0; p < n_patterns; ++p)
        if (entry_of[p] == e) {
          t->out_flat[no].pattern_id = p;
          t->out_flat[no].matched_len = entry_len[e];
          ++no;
        }
    }
  }
  t->out_offsets[nn] = no;
  t->n_out = no;
  free(order), free(renum), free(rows), free(ends);
  free(entry_of), free(entry_src), free(entry_len);
  *out = t;
  return OR_OK;
}

uint32_t or_trie_state_count(const or_trie* t) { return t->state_count; }
const int32_t* or_trie_table(const or_trie* t) { return t->table; }
const uint32_t* or_trie_out_offsets(const or_trie* t) { return t->out_offsets; }
const or_output* or_trie_out_flat(const or_trie* t) { return t->out_flat; }
const uint32_t* or_trie_depth(const or_trie* t) { return t->depth; }

/* ---------------------------------------------------------------------- */
/* pfac_scan (scan.hpp:113-202): one logical worker per start position,    */
/* emit outputs of every visited state, stop at the first missing edge or  */
/* end of text; result sorted by (offset, pattern_id).                     */
/* ---------------------------------------------------------------------- */
static int hit_cmp(const void* a, const void* b) {
  const or_hit* x = a;
  const or_hit* y = b;
  if (x->offset != y->offset) return x->offset < y->offset ? -1 : 1;
  if (x->pattern_id != y->pattern_id)
    return x->pattern_id < y->pattern_id ? -1 : 1;
  return 0;
}

int or_pfac_scan(const uint8_t* text, uint64_t n, const or_trie* t,
                 or_hit** out, uint64_t* n_out) {
  uint64_t cap = 64, nh = 0;
  or_hit* h = malloc(sizeof(or_hit) * cap);
  for (uint64_t i = 0; i < n; ++i) {
    int32_t s = t->table[text[i]]; /* scan.hpp:126 (depth1) */
    if (s < 0) continue;
    uint64_t j = i;
    for (;;) {
      for (uint32_t k = t->out_offsets[s]; k < t->out_offsets[s + 1]; ++k) {
        if (nh == cap) {
          cap *= 2;
          h = realloc(h, sizeof(or_hit) * cap);
          if (!h) return OR_ENOMEM;
        }
        h[nh].offset = i;
        h[nh].pattern_id = t->out_flat[k].pattern_id;
        h[nh].matched_len = t->out_flat[k].matched_len;
        ++nh;
      }
      if (++j >= n) break;                       /* scan.hpp:153 */
      s = t->table[(uint64_t)s * 256 + text[j]]; /* scan.hpp:156 */
      if (s < 0) break;
    }
  }
  qsort(h, nh, sizeof(or_hit), hit_cmp); /* scan.hpp:200 */
  *out = h;
  *n_out = nh;
  return OR_OK;
}

/* ---------------------------------------------------------------------- */
/* naive_scan (scan.hpp:247-260): memcmp of every pattern at every start.  */
/* Emitted as hits with matched_len = full pattern length.                 */
/* ---------------------------------------------------------------------- */
int or_naive_scan(const uint8_t* text, uint64_t n, const uint8_t* bytes,
                  const uint64_t* off, uint32_t n_patterns, or_hit** out,
                  uint64_t* n_out) {
  uint64_t cap = 64, nh = 0;
  or_hit* h = malloc(sizeof(or_hit) * cap);
  for (uint32_t p = 0; p < n_patterns; ++p) {
    uint64_t m = off[p + 1] - off[p];
    if (m == 0 || n < m) continue;
    for (uint64_t i = 0; i + m <= n; ++i)
      if (memcmp(text + i, bytes + off[p], m) == 0) {
        if (nh == cap) {
          cap *= 2;
          h = realloc(h, sizeof(or_hit) * cap);
        }
        h[nh].offset = i;
        h[nh].pattern_id = p;
        h[nh].matched_len = (uint32_t)m;
        ++nh;
      }
  }
  qsort(h, nh, sizeof(or_hit), hit_cmp);
  *out = h;
  *n_out = nh;
  return OR_OK;
}

/* ---------------------------------------------------------------------- */
/* LineIndex::line_of (verify.hpp:40-49): 1 + number of LF in [0, offset]  */
/* with the LF belonging to its own line, i.e. upper_bound over the line   */
/* starts {0} U {i+1 : text[i]==LF}.                                      */
/* ---------------------------------------------------------------------- */
uint64_t or_line_of(const uint8_t* text, uint64_t n, uint64_t offset) {
  uint64_t line = 1;
  for (uint64_t i = 0; i < n && i + 1 <= offset; ++i)
    if (text[i] == '\n') ++line;
  return line;
}

/* ---------------------------------------------------------------------- */
/* verify_hits (verify.hpp:69-105) + assemble_report (verify.hpp:107-117)  */
/* with_lines != 0 fills alert.line (else 0).  Alerts keep (offset,        */
/* rule_id) order.  Returns OR_ELOGIC for a hit past the end of text.      */
/* ---------------------------------------------------------------------- */
static int alert_cmp(const void* a, const void* b) {
  const or_alert* x = a;
  const or_alert* y = b;
  if (x->offset != y->offset) return x->offset < y->offset ? -1 : 1;
  if (x->rule_id != y->rule_id) return x->rule_id < y->rule_id ? -1 : 1;
  return 0;
}

int or_verify_hits(const uint8_t* text, uint64_t n, const or_hit* hits,
                   uint64_t n_hits, const uint8_t* bytes, const uint64_t* off,
                   uint32_t n_patterns, uint64_t prefix_len, int with_lines,
                   or_alert** out, uint64_t* n_out) {
  or_alert* a = malloc(sizeof(or_alert) * (n_hits + 1));
  uint64_t na = 0;
  /* running line counter: hits are not required to be sorted, so compute
   * each line independently when requested */
  for (uint64_t k = 0; k < n_hits; ++k) {
    const or_hit* h = &hits[k];
    if (h->offset + h->matched_len > n) { /* verify.hpp:76-77 */
      free(a);
      return OR_ELOGIC;
    }
    if (h->pattern_id >= n_patterns) {    /* rules.patterns.at() */
      free(a);
      return OR_ELOGIC;
    }
    uint64_t plen = off[h->pattern_id + 1] - off[h->pattern_id];
    int ok;
    if (plen <= prefix_len)
      ok = 1;
    else if (h->offset + plen > n)
      ok = 0;
    else
      ok = memcmp(text + h->offset + h->matched_len,
                  bytes + off[h->pattern_id] + h->matched_len,
                  plen - h->matched_len) == 0;
    if (!ok) continue;
    a[na].offset = h->offset;
    a[na].rule_id = h->pattern_id;
    a[na].pattern_len = (uint32_t)plen;
    a[na].line = with_lines ? or_line_of(text, n, h->offset) : 0;
    ++na;
  }
  qsort(a, na, sizeof(or_alert), alert_cmp); /* verify.hpp:100-103 */
  *out = a;
  *n_out = na;
  return OR_OK;
}

/* ---------------------------------------------------------------------- */
/* KMP (kmp.hpp:25-69)                                                     */
/* ---------------------------------------------------------------------- */
void or_kmp_failure(const uint8_t* p, uint32_t m, uint32_t* table) {
  if (m == 0) return;
  table[0] = 0;
  uint32_t k = 0;
  for (uint32_t i = 1; i < m; ++i) {
    while (k > 0 && p[i] != p[k]) k = table[k - 1];
    if (p[i] == p[k]) ++k;
    table[i] = k;
  }
}

int or_kmp_search(const uint8_t* text, uint64_t n, const uint8_t* p,
                  uint32_t m, const uint32_t* table, uint64_t** out,
                  uint64_t* n_out, uint64_t* comparisons) {
  uint64_t cap = 64, no = 0, cmp = 0;
  uint64_t* o = malloc(sizeof(uint64_t) * cap);
  *out = o;
  *n_out = 0;
  if (m == 0 || n < m) return OR_OK;
  uint64_t i = 0;
  uint32_t j = 0;
  while (i < n) {
    ++cmp;
    if (text[i] == p[j]) {
      ++i;
      ++j;
      if (j == m) {
        if (no == cap) {
          cap *= 2;
          o = realloc(o, sizeof(uint64_t) * cap);
        }
        o[no++] = i - m;
        j = table[m - 1];
      }
    } else if (j > 0) {
      j = table[j - 1];
    } else {
      ++i;
    }
  }
  if (comparisons) *comparisons += cmp;
  *out = o;
  *n_out = no;
  return OR_OK;
}

void or_free(void* p) { free(p); }
