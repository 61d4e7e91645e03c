// glop_kernels.cuh -- sm_100a device code for the GLoP matching path.
//
//   pfac_warp_kernel  K1  PFAC scan (scan.hpp:113-202), two variants:
//                         FILTERED: sampled q-gram filter + 8-byte prefix
//                         bitmap in shared memory, then the trie walk only for
//                         survivors (GPU analogue of RootJump, scan.hpp:81-108)
//                         DIRECT:   one thread per start byte, literal walk
//   seg_reduce / seg_gather  K2  deterministic (offset, pattern_id) order
//                         (scan.hpp:197-201) without a global sort
//   verify_*          K3  stage-2 suffix check (verify.hpp:69-105)
//   (K4 KMP: kmp.cuh; the 8-byte-prefix PFAC fast path: pfac8.cuh)
//   gen_syslog_kernel     synthetic corpus (bench input, not the path)
//
// Text is streamed HBM -> shared memory with 1-D TMA bulk copies
// (cp.async.bulk ... mbarrier::complete_tx) into a ring of stages; one
// persistent CTA per SM walks its tiles round-robin.
#pragma once
#include <stdint.h>

#include "corpus.h"
#include "payload.h"

namespace glop {

constexpr uint32_t kTile = 4096;            // owned start positions per tile
constexpr uint32_t kHalo = 64;              // bytes past the tile kept in smem
constexpr uint32_t kStageBytes = kTile + kHalo + 16;  // +16: alignment slack
constexpr uint32_t kDmaskBits = 15;         // level-1 q-gram d-mask: 2^15 buckets
constexpr uint32_t kDmaskBytes = 1u << kDmaskBits;
constexpr uint32_t kBm2Log2 = 18;
constexpr uint32_t kBm2Bits = 1u << kBm2Log2;  // level-2 prefix bitmap
constexpr uint32_t kBm2Bytes = kBm2Bits / 8;

struct JumpEntry;
struct DevTrie {
  const uint8_t* cls;       // 256 byte -> class
  const void* table;        // Q x C entries, 0 = no edge
  const uint32_t* out_off;  // Q + 1
  const uint32_t* out_pid;  // flat output pattern ids
  const uint32_t* pid_len;  // pattern id -> matched_len
  const uint8_t* dmask;     // kDmaskBytes
  const uint32_t* bm2;      // kBm2Bits / 32 words
  const uint32_t* bm2_8;    // pfac8's level-2 bitmap (kP8Bm2Log2 bits, see pfac8.cuh)
  const JumpEntry* jump;    // open-addressed J-byte jump table
  const uint8_t* dmask8;    // pfac8 level-1 d-masks (lmin >= 8), 2^15 bytes
  uint32_t Q, C, lmin, lmax, q, stride;
  uint32_t table_bytes;     // padded to 16
  uint32_t jump_depth, jump_cap_log2, jump_bytes;
};

// Device twin of glop_hit / logtrawl::Hit (scan.hpp:31-41): 16 bytes.
struct DevHit {
  unsigned long long offset;
  uint32_t pid, len;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// Shared-window address forms (u32), for loops that keep the addresses in
// registers instead of converting generic pointers on every call.
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx_a(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_a(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_g2s_a(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
// TMA prefetch of global [src, src + bytes) into L2 (16-byte aligned, size a
// multiple of 16): memory-level parallelism without shared memory
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ------------------------------------------------------------------ hashing
// Level-1 bucket of a q-gram packed little-endian (q <= 4); q = 1 is exact.
__host__ __device__ __forceinline__ uint32_t qgram_bucket(uint32_t g, uint32_t q) {
  return q == 1 ? g : ((g * 0x9E3779B1u) >> (32 - kDmaskBits));
}
// Level-2 bit of an (up to) 8-byte prefix packed little-endian (lo, hi
// 32-bit halves): two 32-bit multiplies, cheaper than a 64-bit one on the SM.
__host__ __device__ __forceinline__ uint32_t prefix_hash32(uint32_t lo, uint32_t hi) {
  return (lo * 0x9E3779B1u) ^ (hi * 0x85EBCA77u);
}
__host__ __device__ __forceinline__ uint32_t prefix_bit32(uint32_t lo, uint32_t hi) {
  return prefix_hash32(lo, hi) >> (32 - kBm2Log2);
}
__host__ __device__ __forceinline__ uint32_t prefix_bit(unsigned long long key) {
  return prefix_bit32((uint32_t)key, (uint32_t)(key >> 32));
}
// Second level-2 bit of a prefix (PREFIX8 kernel, large prefix sets): the top
// bits of a remultiplied 32-bit hash, independent of prefix_bit's slice.
__host__ __device__ __forceinline__ uint32_t prefix_hash2(uint32_t x) { return x * 0x2C1B3C6Du; }
__host__ __device__ __forceinline__ uint32_t prefix_bit2(unsigned long long key) {
  return prefix_hash2(prefix_hash32((uint32_t)key, (uint32_t)(key >> 32))) >> (32 - kBm2Log2);
}
__host__ __device__ __forceinline__ unsigned long long low_bytes_mask(uint32_t k) {
  return k >= 8 ? ~0ull : ((1ull << (8 * k)) - 1);
}

// ------------------------------------------------------------------ tile ring
// Window of tile t in "aligned" coordinates: A = text - a, a = text & 15.
// Stage bytes [0, kStageBytes) hold A[t*kTile, t*kTile + kStageBytes) clipped
// to the text; text position x lives at win[x + a - t*kTile].
struct Ring {
  uint8_t* stages;
  uint64_t* bars;
  const uint8_t* A;
  uint32_t a;
  unsigned long long n;

  __device__ void issue(int stage, uint32_t t) const {  // one thread
    issue_to(stages + (size_t)stage * kStageBytes, &bars[stage], t);
  }
  __device__ void issue_to(uint8_t* dst, uint64_t* bar, uint32_t t) const {  // one thread
    const unsigned long long lo = (unsigned long long)t * kTile;
    const unsigned long long hi = lo + kStageBytes;
    const unsigned long long vlo = lo > a ? lo : a;               // valid data
    const unsigned long long vhi = hi < a + n ? hi : a + n;
    unsigned long long tlo = (vlo + 15) & ~15ull, thi = vhi & ~15ull;
    if (thi < tlo) thi = tlo;
    for (unsigned long long x = vlo; x < tlo && x < vhi; ++x) dst[x - lo] = A[x];
    for (unsigned long long x = thi > vlo ? thi : vlo; x < vhi; ++x) dst[x - lo] = A[x];
    if (thi > tlo) {
      mbar_arrive_tx(bar, (uint32_t)(thi - tlo));
      bulk_g2s(dst + (tlo - lo), A + tlo, (uint32_t)(thi - tlo), bar);
    } else {
      mbar_arrive(bar);
    }
  }
};

// Unaligned little-endian loads from a stage window (idx + 8 < kStageBytes).
__device__ __forceinline__ uint32_t win_u32(const uint8_t* win, uint32_t idx) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(win + (idx & ~3u));
  return __funnelshift_r(w[0], w[1], (idx & 3u) * 8);
}
__device__ __forceinline__ unsigned long long win_u64(const uint8_t* win, uint32_t idx) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(win + (idx & ~3u));
  const uint32_t sh = (idx & 3u) * 8;
  uint32_t w0 = w[0], w1 = w[1], w2 = w[2];
  return (unsigned long long)__funnelshift_r(w0, w1, sh) |
         ((unsigned long long)__funnelshift_r(w1, w2, sh) << 32);
}

template <typename Entry>
struct EntryTraits;
template <>
struct EntryTraits<uint16_t> {
  static constexpr uint32_t kFlag = 0x8000u, kMask = 0x7FFFu;
};
template <>
struct EntryTraits<uint32_t> {
  static constexpr uint32_t kFlag = 0x80000000u, kMask = 0x7FFFFFFFu;
};

// ------------------------------------------------------------------ K1 PFAC
// Shared-memory layout (byte offsets), computed on the host per automaton.
struct PfacLayout {
  uint32_t bars, cls, misc, keys, queue, cand, dmask, bm2, hash, table, total;
};

__host__ __device__ inline uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }

// Jump-table entry: the trie state reached by a J-byte root path
// (J = min(lmin, 8)), generalising the reference's depth-1/depth-2 RootJump
// (scan.hpp:81-108) to J levels.  state+1 in `state1` (0 = empty slot); `out`
// is the single output pattern id of that state (< kOutList), kOutNone,
// kOutList | (n - 1) << 24 | o for n <= 127 ids at out_pid[o, o + n) (one
// dependent load less than the state's CSR bounds), or kOutMany (the CSR
// list of the state: lists that do not fit the encoding).
struct JumpEntry {
  unsigned long long key;
  uint32_t state1;
  uint32_t out;
};
constexpr uint32_t kOutNone = 0xFFFFFFFFu, kOutMany = 0xFFFFFFFEu, kOutList = 0x80000000u;
__host__ __device__ __forceinline__ uint32_t jump_out(const uint32_t* pid, uint32_t o, uint32_t n) {
  if (n == 0) return kOutNone;
  if (n == 1) return pid[o] < kOutList ? pid[o] : kOutMany;
  return n <= 127 && o < (1u << 24) ? kOutList | (n - 1) << 24 | o : kOutMany;
}

__host__ __device__ __forceinline__ uint32_t jump_slot(unsigned long long key, uint32_t cap_log2) {
  return (uint32_t)((key * 0xD6E8FEB86659FD93ull) >> (64 - cap_log2));
}

// ------------------------------------------------------------------ K1 (per-warp pipelines)
// Sixteen warps per CTA, one CTA per SM.  The CTA takes a contiguous range of
// 4 KB tiles; each warp grabs tiles from it (shared-memory counter) and
// double-buffers them privately: lane 0 issues the TMA bulk copy of the next
// tile into the warp's idle buffer (own mbarrier) while the warp scans the
// current one.  No two warps ever wait for each other.  A warp runs its tile
// end to end: q-gram filter, candidate queue, exact check, ordering of its
// hits, write-out into its private staging region, and one directory record
// per tile.
constexpr int kConsumerWarps = 16;
constexpr int kWarpKernelThreads = kConsumerWarps * 32;
constexpr int kWBuf = 2;           // private tile buffers per warp (double buffering)
constexpr uint32_t kWQueue = 128;  // per-warp filter survivors
constexpr uint32_t kWHits = 64;    // per-warp hit keys of one drain batch (smem)
constexpr uint32_t kWCand = 256;   // per-warp candidates of one drain batch (32 x 8)

struct SegDir {
  uint32_t cursor;  // offset inside the producing warp's staging region
  uint32_t count;
  uint32_t region;  // producing warp (global id)
  uint32_t pad;
};

struct WarpScanParams {
  const uint8_t* text;
  unsigned long long n, own, base;
  uint32_t num_tiles;
  uint32_t num_units;            // unused (per-CTA count derived in-kernel)
  int mode;                      // 0 ordered staging; 1 global keys
  DevHit* staging;
  unsigned long long region;     // staging records per (CTA, warp) region
  SegDir* dir;                   // one record per tile
  unsigned long long* g_count;   // [0] total hits, [1] flags, [2] max region use
  unsigned long long* keys;      // mode 1
  unsigned long long keys_cap;
};

// hash_bytes > 0: jump table in shared memory; otherwise it stays in global
// memory behind the level-2 bitmap kept in shared memory.
__host__ __device__ inline PfacLayout make_warp_layout(bool filter, uint32_t hash_bytes, uint32_t table_bytes) {
  PfacLayout L;
  uint32_t o = kConsumerWarps * kWBuf * kStageBytes;  // private tile buffers
  L.bars = o; o += kConsumerWarps * kWBuf * 8;
  L.cls = o; o += 256;
  L.misc = o; o += align16((kConsumerWarps + 1) * 4);
  L.keys = o; o += kConsumerWarps * kWHits * 8;
  L.queue = o; o += filter ? kConsumerWarps * kWQueue * 4 : 0;
  L.cand = o; o += filter ? kConsumerWarps * kWCand * 2 : 0;
  L.dmask = o; o += filter ? kDmaskBytes : 0;
  L.bm2 = o; o += filter ? kBm2Bytes : 0;
  o = align16(o);
  L.hash = o; o += filter ? hash_bytes : 0;
  o = align16(o);
  L.table = o; o += table_bytes;
  L.total = o;
  return L;
}

// Ascending sort of keys[0, n), n <= 64, by one warp (smem bitonic).
__device__ __forceinline__ void warp_sort_keys(unsigned long long* keys, uint32_t n, uint32_t lane) {
  if (n <= 1) return;
  uint32_t P = 2;
  while (P < n) P <<= 1;
  for (uint32_t x = n + lane; x < P; x += 32) keys[x] = ~0ull;
  __syncwarp();
  for (uint32_t k = 2; k <= P; k <<= 1)
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t x = lane; x < P; x += 32) {
        const uint32_t y = x ^ j;
        if (y > x) {
          const unsigned long long u = keys[x], v = keys[y];
          if ((u > v) == ((x & k) == 0)) keys[x] = v, keys[y] = u;
        }
      }
      __syncwarp();
    }
}

// kS: compile-time sampling stride (0 = runtime tr.stride; 5 = the 8-byte
// prefix case, q = 4).
template <bool kFilter, bool kSmemTable, bool kSmemHash, typename Entry, uint32_t kS>
__global__ void __launch_bounds__(kWarpKernelThreads, 1)
    pfac_warp_kernel(const DevTrie tr, const WarpScanParams p, const PfacLayout L) {
  using ET = EntryTraits<Entry>;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint8_t* s_cls = smem + L.cls;
  const uint8_t* s_dmask = smem + L.dmask;
  const uint32_t* s_bm2 = reinterpret_cast<const uint32_t*>(smem + L.bm2);
  const JumpEntry* H = kSmemHash ? reinterpret_cast<const JumpEntry*>(smem + L.hash) : tr.jump;
  const Entry* T = kSmemTable ? reinterpret_cast<const Entry*>(smem + L.table) : reinterpret_cast<const Entry*>(tr.table);
  // s_misc: [0, kConsumerWarps) per-warp hit counters, [kConsumerWarps] next tile
  uint32_t* s_misc = reinterpret_cast<uint32_t*>(smem + L.misc);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars) + warp * kWBuf;
  uint8_t* bufs = smem + (size_t)warp * kWBuf * kStageBytes;
  // this CTA's contiguous range of tiles [t_begin, t_end)
  const uint32_t per = (p.num_tiles + gridDim.x - 1) / gridDim.x;
  const uint32_t t_begin = min(blockIdx.x * per, p.num_tiles), t_end = min(t_begin + per, p.num_tiles);

  // ---- stage the automaton (all warps), init barriers
  {
    auto copy = [&](uint32_t off, const void* src, uint32_t bytes) {
      const uint4* s = reinterpret_cast<const uint4*>(src);
      uint4* d = reinterpret_cast<uint4*>(smem + off);
      for (uint32_t i = tid; i < bytes / 16; i += kWarpKernelThreads) d[i] = s[i];
    };
    copy(L.cls, tr.cls, 256);
    if (kFilter) {
      copy(L.dmask, tr.dmask, kDmaskBytes);
      copy(L.bm2, tr.bm2, kBm2Bytes);
      if (kSmemHash) copy(L.hash, tr.jump, tr.jump_bytes);
    }
    if (kSmemTable) copy(L.table, tr.table, tr.table_bytes);
    if (tid <= kConsumerWarps) s_misc[tid] = tid < kConsumerWarps ? 0 : t_begin + kConsumerWarps * kWBuf;
    if (lane < kWBuf) mbar_init(&bars[lane], 1);
    if (tid == 0) fence_mbar_init();
  }
  __syncthreads();
  const uint32_t a = (uint32_t)((uintptr_t)p.text & 15);
  Ring ring{nullptr, nullptr, p.text - a, a, p.n};

  // Each warp double-buffers its own tiles: lane 0 keeps kWBuf - 1 tiles in
  // flight (TMA bulk copies into the warp's private buffers) while the warp
  // scans the current one.  Tiles come from the CTA's range: the first
  // kWBuf per warp statically, then the next free one.
  uint32_t pend[kWBuf];  // tile held / in flight per buffer (t_end = none)
#pragma unroll
  for (uint32_t b = 0; b < kWBuf; ++b) {
    pend[b] = t_begin + warp * kWBuf + b;
    if (pend[b] >= t_end) pend[b] = t_end;
    if (lane == 0 && pend[b] < t_end) ring.issue_to(bufs + b * kStageBytes, &bars[b], pend[b]);
  }
  uint32_t use[kWBuf] = {};  // completed uses per buffer (mbarrier phase)

  uint32_t* q = reinterpret_cast<uint32_t*>(smem + L.queue) + warp * kWQueue;
  uint16_t* cand = reinterpret_cast<uint16_t*>(smem + L.cand) + warp * kWCand;
  uint32_t* s_nh = s_misc;
  unsigned long long* hk = reinterpret_cast<unsigned long long*>(smem + L.keys) + warp * kWHits;
  const uint32_t gw = blockIdx.x * kConsumerWarps + warp;  // staging region of this warp
  const unsigned long long region_base = (unsigned long long)gw * p.region;
  uint32_t cursor = 0;  // records written into this warp's staging region
  const uint32_t qg = tr.q, S = kS ? kS : tr.stride, lmin = tr.lmin, J = tr.jump_depth;
  const uint32_t cap_log2 = tr.jump_cap_log2;
  const uint32_t qmask = qg >= 4 ? 0xFFFFFFFFu : ((1u << (8 * qg)) - 1);
  const unsigned long long jmask = low_bytes_mask(J);
  const uint32_t hmask = (1u << cap_log2) - 1;
  const uint32_t lmax = tr.lmax, C = tr.C;
  const unsigned long long own_end = p.own + a, n_end = p.n + a;  // aligned coordinates

  for (uint32_t b = 0;; b = (b + 1 == kWBuf) ? 0 : b + 1) {
    const uint32_t t = pend[b];
    if (t >= t_end) break;
    mbar_wait(&bars[b], use[b] & 1);
    ++use[b];
    // Window coordinates y: sb[y] = aligned byte A[t*kTile + y] = text
    // position t*kTile + y - a, so chunks are word aligned.
    const uint8_t* sb = bufs + b * kStageBytes;
    const uint32_t* sw = reinterpret_cast<const uint32_t*>(sb);
    const unsigned long long tA = (unsigned long long)t * kTile;
    const uint32_t s_hi = (uint32_t)min(own_end - tA, (unsigned long long)kTile);
    const uint32_t avail = (uint32_t)min(n_end - tA, 0x7FFFFFFFull);  // valid bytes y < avail
    const uint32_t s_lo = 0;
    const uint32_t lo = t == 0 ? a : 0;  // tile 0 starts at text offset 0
    const unsigned long long off0 = p.base + tA - a;  // text offset of window position 0
    uint32_t seg_n = 0;  // hits of this tile written so far (warp-uniform)

    auto emit = [&](uint32_t y, uint32_t pid) {
      if (p.mode == 0) {
        const uint32_t slot = atomicAdd(&s_nh[warp], 1u);
        if (slot < kWHits) hk[slot] = ((unsigned long long)(y - s_lo) << 40) | pid;
      } else {
        const unsigned long long slot = atomicAdd(p.g_count + 3, 1ull);
        if (slot < p.keys_cap) p.keys[slot] = ((off0 + y) << 24) | pid;
      }
    };
    // sorts the buffered batch and appends it to the warp's staging region;
    // false if the batch overflowed the buffer (nothing written)
    auto flush = [&]() -> bool {
      __syncwarp();
      const uint32_t nb = s_nh[warp];
      if (p.mode != 0 || nb == 0) return true;
      if (nb > kWHits) return false;
      warp_sort_keys(hk, nb, lane);
      if (cursor + seg_n + nb <= p.region)
        for (uint32_t h = lane; h < nb; h += 32) {
          const unsigned long long key = hk[h];
          const uint32_t pid = (uint32_t)(key & 0xFFFFFFFFFFull);
          DevHit out;
          out.offset = off0 + s_lo + (key >> 40);
          out.pid = pid;
          out.len = __ldg(tr.pid_len + pid);
          p.staging[region_base + cursor + seg_n + h] = out;
        }
      seg_n += nb;
      __syncwarp();
      if (lane == 0) s_nh[warp] = 0;
      __syncwarp();
      return true;
    };
    auto discard = [&]() {  // drop the buffered batch (it will be redone)
      __syncwarp();
      if (lane == 0) s_nh[warp] = 0;
      __syncwarp();
    };
    // a single start produced more hits than the buffer holds: count them
    // (so the host can size the exact fallback) and flag the scan
    auto overflow = [&]() {
      __syncwarp();
      if (lane == 0) {
        atomicAdd(p.g_count, (unsigned long long)s_nh[warp]);
        atomicOr(reinterpret_cast<unsigned int*>(p.g_count + 1), 1u);
        s_nh[warp] = 0;
      }
      __syncwarp();
    };
    auto tbyte = [&](uint32_t y) -> uint32_t {  // y < avail
      return y < kStageBytes ? sb[y] : __ldg(p.text + (tA + y - a));
    };
    auto emit_state = [&](uint32_t y, uint32_t st) {
      for (uint32_t o = __ldg(tr.out_off + st), oe = __ldg(tr.out_off + st + 1); o < oe; ++o)
        emit(y, __ldg(tr.out_pid + o));
    };
    // PFAC walk (scan.hpp:142-168) from state st at window byte j
    auto walk = [&](uint32_t y, uint32_t st, uint32_t j) {
      for (; j < avail; ++j) {
        const uint32_t c = s_cls[tbyte(j)];
        const uint32_t e = kSmemTable ? (uint32_t)T[st * C + c] : (uint32_t)__ldg(T + st * C + c);
        if (!e) break;
        st = e & ET::kMask;
        if (e & ET::kFlag) emit_state(y, st);
      }
    };

#ifdef GLOP_EXP_NOWORK
    if (false) {
#else
    if (kFilter) {
#endif
      // level-2 test of candidate start y: the J-byte prefix must hit the
      // prefix bitmap; survivors probe the jump table (exact, generalised
      // RootJump, scan.hpp:81-108) and walk the remaining levels.
      auto check = [&](uint32_t y) {
        const unsigned long long key = win_u64(sb, y) & jmask;
        const uint32_t bit = prefix_bit(key);
        if (!((s_bm2[bit >> 5] >> (bit & 31)) & 1u)) return;
        for (uint32_t h = jump_slot(key, cap_log2);; h = (h + 1) & hmask) {
          const JumpEntry e = H[h];
          if (!e.state1) return;
          if (e.key != key) continue;
          const uint32_t st = e.state1 - 1;
          if (e.out != kOutNone) {
            if (e.out < kOutList) emit(y, e.out);
            else if (e.out == kOutMany) emit_state(y, st);
            else
              for (uint32_t o = e.out & 0xFFFFFFu, oe = o + ((e.out >> 24) & 0x7Fu) + 1; o < oe; ++o)
                emit(y, __ldg(tr.out_pid + o));
          }
          if (lmax > J) walk(y, st, y + J);
          return;
        }
      };
      // Queue entries (P << 8) | dmask are in increasing P order, so the
      // hits of consecutive 32-entry batches are ordered batch to batch:
      // each batch is expanded into candidates (one per set d bit), checked
      // 32 at a time, then sorted and flushed.  A batch that overflows the
      // hit buffer is redone one entry at a time.
      auto drain = [&](uint32_t qn) {
#ifdef GLOP_EXP_NODRAIN
        qn = 0;
#endif
        __syncwarp();  // the queue entries other lanes pushed are visible (racecheck)
        for (uint32_t e0 = 0; e0 < qn; e0 += 32) {
          const uint32_t v = e0 + lane < qn ? q[e0 + lane] : 0u;
          const uint32_t c = __popc(v & 0xFFu);
          uint32_t pre = c;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(0xffffffffu, pre, o);
            if (lane >= (uint32_t)o) pre += x;
          }
          const uint32_t tot = __shfl_sync(0xffffffffu, pre, 31);
          {
            uint32_t at = pre - c, dm = v & 0xFFu;
            while (dm) {
              const uint32_t d = __ffs(dm) - 1;
              dm &= dm - 1;
              cand[at++] = (uint16_t)((v >> 8) - d);
            }
          }
          __syncwarp();
          for (uint32_t c0 = 0; c0 < tot; c0 += 32)
            if (c0 + lane < tot) check(cand[c0 + lane]);
          if (!flush()) {
            discard();
            for (uint32_t j = 0; j < 32 && e0 + j < qn; ++j) {
              if (lane == j) {
                uint32_t dm = v & 0xFFu;
                while (dm) {
                  const uint32_t d = __ffs(dm) - 1;
                  dm &= dm - 1;
                  check((v >> 8) - d);
                }
              }
              if (!flush()) overflow();
            }
          }
        }
      };
      auto bucket = [&](uint32_t g) -> uint32_t {
        return kS ? ((g * 0x9E3779B1u) >> (32 - kDmaskBits)) : qgram_bucket(g & qmask, qg);  // kS > 0: q = 4
      };
      // d-mask of sampled position P restricted to lo <= P - d < s_hi,
      // P - d + lmin <= avail, P + q <= avail
      auto probe_edge = [&](uint32_t P) -> uint32_t {
        if (P + qg > avail) return 0;
        uint32_t dm = s_dmask[bucket(win_u32(sb, P))];
        if (dm) {
          if (P < lo) return 0;
          if (P - lo < 7) dm &= (2u << (P - lo)) - 1;
          if (P >= s_hi) dm &= ~((2u << min(P - s_hi, 7u)) - 1);
          if (P + lmin > avail) dm = P + lmin - avail > 7 ? 0 : dm & ~((1u << (P + lmin - avail)) - 1);
        }
        return dm;
      };
      uint32_t qn = 0;
      auto push = [&](uint32_t m, uint32_t dm) {
        const uint32_t bal = __ballot_sync(0xffffffffu, dm != 0);
        if (bal) {
          if (qn + 32 > kWQueue) {
            drain(qn);
            qn = 0;
          }
          if (dm) q[qn + __popc(bal & ((1u << lane) - 1))] = ((m * S) << 8) | dm;
          qn += __popc(bal);
        }
      };
      // sampled positions P = m*S whose candidates P - d (d < S) can start in
      // [lo, s_hi): m in [ceil(lo/S), ceil((s_hi+S-1)/S)); positions in
      // [safe_lo, safe_hi) need no range masks on a full interior tile
      const bool fast = lo == 0 && s_hi == kTile && avail >= kTile + 16;
      const uint32_t m1 = s_hi > lo ? (s_hi + 2 * S - 2) / S : 0;
      uint32_t base = s_hi > lo ? (lo + S - 1) / S : m1;
      if (fast) {
        const uint32_t safe_lo = (7 + S - 1) / S, safe_hi = kTile / S;
        // leading edge plus alignment to a multiple of 4 positions, masked
        const uint32_t ia = (safe_lo + 3) & ~3u;
        {
          const uint32_t m = base + lane;
          uint32_t dm = 0;
          if (m < ia) dm = m < safe_lo ? probe_edge(m * S) : s_dmask[bucket(win_u32(sb, m * S))];
          push(m, dm);
        }
        base = ia;
        if (kS) {
          // 4 consecutive sampled positions per lane from word-aligned,
          // conflict-free loads; one vote per 128 positions
          constexpr uint32_t kW = (3 * kS + 4 + 3) / 4;
          for (; base + 128 <= safe_hi; base += 128) {
            const uint32_t B = (base + 4 * lane) * kS;  // multiple of 4
            uint32_t w[kW + 1];
#pragma unroll
            for (uint32_t i = 0; i <= kW; ++i) w[i] = sw[B / 4 + i];
            uint32_t dm[4];
#pragma unroll
            for (uint32_t v = 0; v < 4; ++v) {
              const uint32_t o = v * kS;
              const uint32_t g = (o & 3) ? __funnelshift_r(w[o / 4], w[o / 4 + 1], 8 * (o & 3)) : w[o / 4];
              dm[v] = s_dmask[bucket(g)];
            }
            const uint32_t cnt = (dm[0] != 0) + (dm[1] != 0) + (dm[2] != 0) + (dm[3] != 0);
            if (__ballot_sync(0xffffffffu, cnt != 0)) {
              // queue in position order (lane-major): exclusive warp scan
              uint32_t pre = cnt;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const uint32_t x = __shfl_up_sync(0xffffffffu, pre, o);
                if (lane >= (uint32_t)o) pre += x;
              }
              const uint32_t tot = __shfl_sync(0xffffffffu, pre, 31);
              if (qn + tot > kWQueue) {
                drain(qn);
                qn = 0;
              }
              uint32_t at = qn + pre - cnt;
#pragma unroll
              for (uint32_t v = 0; v < 4; ++v)
                if (dm[v]) q[at++] = ((B + v * kS) << 8) | dm[v];
              qn += tot;
              __syncwarp();
            }
          }
        }
        for (; base + 32 <= safe_hi; base += 32)
          push(base + lane, s_dmask[bucket(win_u32(sb, (base + lane) * S))]);
      }
      for (; base < m1; base += 32) {
        const uint32_t m = base + lane;
        push(m, m < m1 ? probe_edge(m * S) : 0u);
      }
      drain(qn);
    } else if (!kFilter) {
      // DIRECT: one lane per start byte
      for (uint32_t y0 = lo; y0 < s_hi; y0 += 32) {
        if (y0 + lane < s_hi) walk(y0 + lane, 0u, y0 + lane);
        if (!flush()) {  // dense batch: one start at a time
          discard();
          for (uint32_t j = 0; j < 32 && y0 + j < s_hi; ++j) {
            if (lane == j) walk(y0 + j, 0u, y0 + j);
            if (!flush()) overflow();
          }
        }
      }
    }
    // buffer b is free: refill it with the next tile of the CTA's range
    __syncwarp();
    uint32_t nxt = t_end;
    if (lane == 0) {
      if (p.mode == 0) {
        p.dir[t] = SegDir{cursor, seg_n, gw, 0};
        if (seg_n) atomicAdd(p.g_count, (unsigned long long)seg_n);
      }
      nxt = atomicAdd(&s_misc[kConsumerWarps], 1u);
      if (nxt < t_end) {
        fence_proxy_async();
        ring.issue_to(bufs + b * kStageBytes, &bars[b], nxt);
      } else {
        nxt = t_end;
      }
    }
    pend[b] = __shfl_sync(0xffffffffu, nxt, 0);
    cursor += seg_n;
  }
  if (p.mode == 0 && lane == 0 && cursor) atomicMax(p.g_count + 2, (unsigned long long)cursor);
}

// ---- segment directory -> ordered output
// Pass 1: per-block sums of segment counts (kSegPerBlock segments per block).
constexpr uint32_t kSegPerThread = 8;
constexpr uint32_t kSegPerBlock = 1024 * kSegPerThread;

__global__ void __launch_bounds__(1024) seg_reduce_kernel(const SegDir* dir, unsigned long long nseg,
                                                          uint32_t* block_sums) {
  __shared__ uint32_t ws[32];
  const unsigned long long b = (unsigned long long)blockIdx.x * kSegPerBlock + threadIdx.x * kSegPerThread;
  uint32_t s = 0;
  for (uint32_t i = 0; i < kSegPerThread; ++i)
    if (b + i < nseg) s += dir[b + i].count;
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t v = ws[threadIdx.x];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = v;
  }
}

// Pass 3 (after block_prefix_kernel over block sums): per-block exclusive scan
// of segment counts, then each thread copies its segments' records.
template <typename Rec>
__global__ void __launch_bounds__(1024) seg_gather_kernel(const SegDir* dir, unsigned long long nseg,
                                                          const unsigned long long* block_prefix,
                                                          uint32_t grid, unsigned long long region,
                                                          const Rec* staging, Rec* out) {
  __shared__ uint32_t ws[32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const unsigned long long b = (unsigned long long)blockIdx.x * kSegPerBlock + tid * kSegPerThread;
  uint32_t c[kSegPerThread], s = 0;
  for (uint32_t i = 0; i < kSegPerThread; ++i) {
    c[i] = b + i < nseg ? dir[b + i].count : 0;
    s += c[i];
  }
  uint32_t incl = s;  // warp inclusive scan
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) ws[w] = incl;
  __syncthreads();
  if (w == 0) {
    uint32_t v = ws[lane], iv = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, iv, o);
      if (lane >= o) iv += u;
    }
    ws[lane] = iv - v;
  }
  __syncthreads();
  unsigned long long dst = block_prefix[blockIdx.x] + ws[w] + incl - s;
  for (uint32_t i = 0; i < kSegPerThread; ++i) {
    if (!c[i]) continue;
    const unsigned long long seg = b + i;
    const unsigned long long src = (unsigned long long)dir[seg].region * region + dir[seg].cursor;
    for (uint32_t h = 0; h < c[i]; ++h) out[dst + h] = staging[src + h];
    dst += c[i];
  }
}

// Global-key fallback: sorted (offset << 24 | pid) keys -> hits.
__global__ void keys_to_hits_kernel(const unsigned long long* keys, unsigned long long n,
                                    const uint32_t* pid_len, DevHit* out) {
  for (unsigned long long h = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; h < n;
       h += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[h];
    DevHit r;
    r.offset = k >> 24;
    r.pid = (uint32_t)(k & 0xFFFFFF);
    r.len = pid_len[r.pid];
    out[h] = r;
  }
}

// ------------------------------------------------------------------ K3 verify
struct DevRules {
  const uint8_t* bytes;
  const unsigned long long* off;
  uint32_t n_patterns;
  unsigned long long prefix_len;
};

struct DevAlert {
  unsigned long long offset;
  uint32_t rule_id, pattern_len;
};

constexpr int kVerifyBlock = 1024;

// Pass 1: keep flags, per-block keep counts, error / order flags.
// text holds global offsets [base, base + n).
__global__ void __launch_bounds__(kVerifyBlock) verify_flags_kernel(
    const DevRules r, const uint8_t* text, unsigned long long base, unsigned long long n, const DevHit* hits,
    unsigned long long n_hits, uint8_t* keep, uint32_t* block_counts, unsigned int* flags) {
  __shared__ uint32_t s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const unsigned long long h = blockIdx.x * (unsigned long long)kVerifyBlock + threadIdx.x;
  uint32_t ok = 0;
  if (h < n_hits) {
    const DevHit x = hits[h];
    if (x.offset < base || x.offset + x.len > base + n || x.pid >= r.n_patterns) {  // verify.hpp:76-77, .at()
      atomicOr(flags, 1u);
    } else {
      const unsigned long long pb = r.off[x.pid], plen = r.off[x.pid + 1] - pb;
      if (plen <= r.prefix_len) {
        ok = 1;
      } else if (x.offset + plen > base + n) {
        ok = 0;
      } else {
        ok = 1;
        for (unsigned long long k = x.len; k < plen; ++k)
          if (text[x.offset - base + k] != r.bytes[pb + k]) {
            ok = 0;
            break;
          }
      }
    }
    if (h + 1 < n_hits) {
      const DevHit y = hits[h + 1];
      if (y.offset < x.offset || (y.offset == x.offset && y.pid < x.pid)) atomicOr(flags, 2u);
    }
    keep[h] = (uint8_t)ok;
  }
  const uint32_t bal = __ballot_sync(0xffffffffu, ok);
  if ((threadIdx.x & 31) == 0 && bal) atomicAdd(&s_cnt, __popc(bal));
  __syncthreads();
  if (threadIdx.x == 0) block_counts[blockIdx.x] = s_cnt;
}

__global__ void __launch_bounds__(1024) block_prefix_kernel(const uint32_t* counts, uint32_t nb,
                                                            unsigned long long* prefix,
                                                            unsigned long long* total) {
  __shared__ unsigned long long part[1024];
  const uint32_t tid = threadIdx.x;
  const uint32_t per = (nb + 1023) / 1024;
  const uint32_t b = tid * per, e = min(nb, b + per);
  unsigned long long s = 0;
  for (uint32_t i = b; i < e; ++i) s += counts[i];
  part[tid] = s;
  __syncthreads();
  for (uint32_t off = 1; off < 1024; off <<= 1) {
    unsigned long long v = tid >= off ? part[tid - off] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  unsigned long long run = part[tid] - s;
  for (uint32_t i = b; i < e; ++i) {
    prefix[i] = run;
    run += counts[i];
  }
  if (tid == 1023) *total = part[1023];
}

// Pass 2: stable compaction of kept hits into alerts (+ per-pattern counts).
__global__ void __launch_bounds__(kVerifyBlock) verify_scatter_kernel(
    const DevRules r, const DevHit* hits, unsigned long long n_hits, const uint8_t* keep,
    const unsigned long long* block_prefix, DevAlert* out, unsigned long long* counts) {
  __shared__ uint32_t warp_base[kVerifyBlock / 32];
  const unsigned long long h = blockIdx.x * (unsigned long long)kVerifyBlock + threadIdx.x;
  const uint32_t ok = h < n_hits ? keep[h] : 0;
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t bal = __ballot_sync(0xffffffffu, ok);
  if (lane == 0) warp_base[w] = __popc(bal);
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (int i = 0; i < kVerifyBlock / 32; ++i) {
      uint32_t c = warp_base[i];
      warp_base[i] = run;
      run += c;
    }
  }
  __syncthreads();
  if (ok) {
    const DevHit x = hits[h];
    const unsigned long long dst =
        block_prefix[blockIdx.x] + warp_base[w] + __popc(bal & ((1u << lane) - 1));
    DevAlert a;
    a.offset = x.offset;
    a.rule_id = x.pid;
    a.pattern_len = (uint32_t)(r.off[x.pid + 1] - r.off[x.pid]);
    out[dst] = a;
    if (counts) atomicAdd(counts + x.pid, 1ull);
  }
}

// Per-pattern alert histogram (the count half of verify_hits' report):
// grid-stride over the alerts into a shared-memory histogram per block,
// then one global atomic per non-empty bin -- instead of one global atomic
// per alert, which serialises on popular patterns.  k <= kHistBins.
constexpr uint32_t kHistBins = 8192;
__global__ void __launch_bounds__(1024) alert_histogram_kernel(const DevAlert* alerts, unsigned long long n,
                                                               uint32_t k, unsigned long long* counts) {
  __shared__ uint32_t h[kHistBins];
  for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    atomicAdd(&h[alerts[i].rule_id], 1u);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < k; i += blockDim.x)
    if (h[i]) atomicAdd(counts + i, (unsigned long long)h[i]);
}

// verify_hits when every pattern is at most prefix_len long (all hits are
// auto-verified, verify.hpp:79-81): one pass converts hits to alerts, checks
// bounds / ids (flag 1, the reference's logic_error) and order (flag 2), and
// builds the per-pattern histogram (shared memory when k <= kHistBins).
__global__ void __launch_bounds__(1024) verify_all_kernel(const DevRules r, unsigned long long base,
                                                          unsigned long long n, const DevHit* hits,
                                                          unsigned long long n_hits, DevAlert* out,
                                                          unsigned long long* counts, unsigned int* flags) {
  __shared__ uint32_t h[kHistBins];
  const bool hist = counts && r.n_patterns <= kHistBins;
  if (hist)
    for (uint32_t i = threadIdx.x; i < r.n_patterns; i += blockDim.x) h[i] = 0;
  __syncthreads();
  unsigned int fl = 0;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n_hits;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const DevHit x = hits[i];
    if (x.offset < base || x.offset + x.len > base + n || x.pid >= r.n_patterns) {
      fl |= 1u;
      continue;
    }
    if (i + 1 < n_hits) {
      const DevHit y = hits[i + 1];
      if (y.offset < x.offset || (y.offset == x.offset && y.pid < x.pid)) fl |= 2u;
    }
    DevAlert a;
    a.offset = x.offset;
    a.rule_id = x.pid;
    a.pattern_len = (uint32_t)(r.off[x.pid + 1] - r.off[x.pid]);
    out[i] = a;
    if (hist) atomicAdd(&h[x.pid], 1u);
    else if (counts) atomicAdd(counts + x.pid, 1ull);
  }
  if (fl) atomicOr(flags, fl);
  __syncthreads();
  if (hist)
    for (uint32_t i = threadIdx.x; i < r.n_patterns; i += blockDim.x)
      if (h[i]) atomicAdd(counts + i, (unsigned long long)h[i]);
}

// Unsorted-input path of verify: alerts <-> (offset << 24 | rule) keys.
__global__ void alerts_to_keys_kernel(const DevAlert* a, unsigned long long n, unsigned long long* keys) {
  for (unsigned long long h = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; h < n;
       h += (unsigned long long)gridDim.x * blockDim.x)
    keys[h] = (a[h].offset << 24) | a[h].rule_id;
}
__global__ void keys_to_alerts_kernel(const unsigned long long* keys, unsigned long long n, const DevRules r,
                                      DevAlert* out) {
  for (unsigned long long h = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; h < n;
       h += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[h];
    DevAlert a;
    a.offset = k >> 24;
    a.rule_id = (uint32_t)(k & 0xFFFFFF);
    a.pattern_len = (uint32_t)(r.off[a.rule_id + 1] - r.off[a.rule_id]);
    out[h] = a;
  }
}

// K4 KMP: see kmp.cuh.

// ------------------------------------------------------------------ corpus
__global__ void gen_syslog_kernel(uint8_t* out, unsigned long long begin, unsigned long long n,
                                  unsigned long long seed) {
  using glop_corpus::kBlock;
  const unsigned long long b0 = begin / kBlock, b1 = (begin + n - 1) / kBlock + 1;
  for (unsigned long long b = b0 + blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; b < b1;
       b += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long s = b * kBlock > begin ? b * kBlock : begin;
    const unsigned long long e = (b + 1) * kBlock < begin + n ? (b + 1) * kBlock : begin + n;
    glop_corpus::gen_block_range(out + (s - begin), seed, b, (uint32_t)(s - b * kBlock),
                                 (uint32_t)(e - b * kBlock));
  }
}

__global__ void gen_payload_kernel(uint8_t* out, unsigned long long begin, unsigned long long n,
                                   unsigned long long seed) {
  using glop_payload::kBlock;
  const unsigned long long b0 = begin / kBlock, b1 = (begin + n - 1) / kBlock + 1;
  for (unsigned long long b = b0 + blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; b < b1;
       b += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long s = b * kBlock > begin ? b * kBlock : begin;
    const unsigned long long e = (b + 1) * kBlock < begin + n ? (b + 1) * kBlock : begin + n;
    glop_payload::gen_block_range(out + (s - begin), seed, b, (uint32_t)(s - b * kBlock),
                                  (uint32_t)(e - b * kBlock));
  }
}

}  // namespace glop
