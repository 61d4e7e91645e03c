// pfac8.cuh -- K1 fast path: PFAC for automata whose outputs all lie at depth
// >= 8 (every pattern prefix has 8 bytes; the north_star's "8-character
// truncated prefixes").  Same result as pfac_scan (scan.hpp:113-202) and the
// general kernel in glop_kernels.cuh, with far fewer instructions per byte:
//
//  * One 768-thread CTA per SM; each of its 24 warps streams a CONTIGUOUS
//    segment of 2 KB tiles through a private double-buffered TMA pipeline
//    (cp.async.bulk + mbarrier).  A warp's hits are therefore produced in text
//    order: its staging region is already sorted, and the final output is the
//    concatenation of the regions in warp order (no per-tile directory).
//  * Level 1, aligned 5-byte grams: every match start c has, for the unique
//    d in 1..4 with c + d = 0 (mod 4), an aligned text word i whose bytes
//    [4i-1, 4i+4) are pattern bytes [d-1, d+4).  A lane owns 16 sample words
//    per tile, 4 consecutive in each 512-byte quarter, read by one
//    conflict-free LDS.128 per quarter (consecutive lanes, consecutive 16 B:
//    the earlier 8-consecutive-words layout was a 2-way bank conflict, and
//    shared-memory wavefronts bound this kernel); each word gets one hashed
//    probe of a 64 KB table: d-mask bytes for small gram sets, single bits
//    (2^19 buckets) above kP8BitsGrams.
//  * Candidate words are compacted in text order into a u16 queue (one
//    packed shuffle scan gives all four quarters' prefixes) and checked 32 per
//    round: the 8-byte key of candidate c = 4i - d is assembled from words
//    i-1, i, i+1 with constant funnel shifts and tested in a 2^18-bit prefix
//    bitmap (one bit per prefix; two above kP8Bloom2Keys prefixes).
//  * Bitmap survivors probe the exact J=8 jump table (generalised RootJump,
//    scan.hpp:81-108) in global memory (L2-resident) and, for patterns longer
//    than 8 bytes, continue the trie walk (scan.hpp:142-168).
//  * Hits are buffered as (offset, id) keys in shared memory and flushed in
//    sorted batches (a lane emits its candidates in ascending offset, so a
//    batch is usually in order already and the warp sort is skipped); a
//    round that overflows the buffer is replayed lane by
//    lane, and a single lane that overflows it flags the exact global-key
//    fallback (radix sort), so any hit density is handled exactly.
#pragma once
#include "glop_kernels.cuh"

namespace glop {

#ifndef GLOP_P8_WARPS
#define GLOP_P8_WARPS 24
#endif
#ifndef GLOP_P8_DMASK_LOG2
#define GLOP_P8_DMASK_LOG2 16
#endif
constexpr int kP8Warps = GLOP_P8_WARPS;
constexpr int kP8Threads = kP8Warps * 32;
constexpr uint32_t kP8Tile = 2048;                 // owned starts per tile (TMA unit)
constexpr uint32_t kP8Stage = kP8Tile + 16;        // + the 4 words after the tile (halo)
constexpr uint32_t kP8Queue = kP8Tile / 4;         // candidate words of one tile, worst case (u16)
constexpr uint32_t kP8Hits = 32;                   // hit keys per warp in smem
// Flush the hit buffer once a round leaves more keys than this (a later round
// that overflows the remaining slots is replayed lane by lane; a single lane
// overflowing them takes the exact global-key fallback).  Higher thresholds
// send DPI lanes with several ids per prefix to that fallback.
#ifndef GLOP_P8_FLUSH_AT
#define GLOP_P8_FLUSH_AT 16
#endif
// L2 prefetch distance: each warp also prefetches (TMA, into L2 only) the
// tiles this many past the two in its shared-memory pipeline
#ifndef GLOP_P8_L2PF
#define GLOP_P8_L2PF 0
#endif
constexpr uint32_t kP8L2Pf = GLOP_P8_L2PF;
#ifndef GLOP_P8_CARRY
#define GLOP_P8_CARRY 1
#endif
#ifndef GLOP_P8_FASTREFILL
#define GLOP_P8_FASTREFILL 1
#endif
constexpr uint32_t kP8DmaskLog2 = GLOP_P8_DMASK_LOG2;
constexpr uint32_t kP8DmaskBytes = 1u << kP8DmaskLog2;  // level-1 d-mask table (shared memory)
// level-2 prefix bitmap of the pfac8 kernel (shared memory): 2^18 bits by
// default; a 2^17-bit map frees 16 KB of shared memory (for more warps) at the
// cost of twice the level-2 false positives (each one an L2 jump-table probe)
#ifndef GLOP_P8_BM2_LOG2
#define GLOP_P8_BM2_LOG2 18
#endif
constexpr uint32_t kP8Bm2Log2 = GLOP_P8_BM2_LOG2;
constexpr uint32_t kP8Bm2Bytes = (1u << kP8Bm2Log2) / 8;

struct P8Layout {
  uint32_t bufs, bars, queue, hits, nh, dmask, bm2, cls, total;
};

__host__ __device__ inline P8Layout make_p8_layout() {
  P8Layout L;
  uint32_t o = 0;
  L.bufs = o; o += kP8Warps * 2 * kP8Stage;
  L.bars = o; o += kP8Warps * 2 * 8;
  L.queue = o; o += kP8Warps * kP8Queue * 2;
  L.hits = o; o += kP8Warps * kP8Hits * 8;
  L.nh = o; o += kP8Warps * 4;
  L.dmask = align16(o); o = L.dmask + kP8DmaskBytes;
  L.bm2 = o; o += kP8Bm2Bytes;
  L.cls = o; o += 256;
  L.total = o;
  return L;
}

struct P8Params {
  const uint8_t* text;
  unsigned long long n, own, base;
  uint32_t num_tiles;
  uint32_t per;                  // tiles per CTA (contiguous range)
  uint32_t sub;                  // tiles per warp segment inside the CTA range
  int mode;                      // 0 ordered staging; 1 global keys
  DevHit* staging;
  unsigned long long region;     // staging records per (CTA, warp)
  unsigned long long* counts;    // hits per (CTA, warp) region
  unsigned long long* g_count;   // [0] total hits, [1] flags, [2] max region use, [3] mode-1 slots
  unsigned long long* keys;      // mode 1
  unsigned long long keys_cap;
  const uint8_t* dmask8;         // 2^16 d-masks (bits 0..3: offsets d = 1..4)
  unsigned long long* zero;      // optional: zeroed by the grid before the scan (the pipeline's per-pattern counts)
  uint32_t nzero;
};

// Level-1 d-mask of an aligned text word (bit d-1: the word may be the
// 5-gram at offset d of some 8-byte prefix), one hashed probe.  A two-hash
// Bloom variant halved the candidate words but doubled the bank-conflicted
// shared-memory probes, which bound the kernel (measured: 3.63 -> 3.55 ms at
// k=1,000 and 2.46 -> 1.97 ms at k=10 without it).  Built by glop_trie_upload.
// Two layouts of the same 64 KB: kBits = false, 2^16 one-byte buckets
// holding the d-mask (bits 0..3); kBits = true, 2^19 one-bit buckets
// ("some offset d may match": the drain tests all four).  Above ~1,000
// distinct grams hash collisions dominate the candidate words and the 8x
// finer bit table wins despite two more instructions per probe (measured:
// k=1,000 2.76 -> 2.60 ms, DPI 10,000 contents 3.40 -> 2.87 ms, syslog
// k=10,000 6.04 -> 4.03 ms; an intermediate 2^17 x 4-bit layout sat between).
// The host picks per automaton (glop_trie_upload: bits above kP8BitsGrams).
constexpr uint32_t kP8BitsGrams = 1024;
// Above this many 8-byte prefixes the 2^18-bit level-2 bitmap passes too many
// (word, d) pairs to the exact L2 probe: set and test a second bit per prefix.
constexpr uint32_t kP8Bloom2Keys = 3000;
// Level-1 probe of sample word i over the 5 bytes [4i-1, 4i+4) -- the
// aligned word `cur` and the top byte of the previous word -- which for a
// match at c = 4i - d (d = 1..4) are pattern bytes [d-1, d+4).  Five bytes
// instead of four cut the candidate words by ~40% on the syslog vocabulary
// set.
//  * bit layouts: the table word is the high half of cur * K (IMAD.HI, a
//    well-mixed hash of the 4 bytes) XORed with the previous word's top byte
//    at bits 8..15 (one PRMT) and masked to a word offset -- one LOP3 does
//    both -- and the bit inside it is cur & 31 (byte 4i; the funnel shift
//    takes its amount straight from `cur`), the second bit of the two-bit
//    layout (cur >> 8) & 31 (byte 4i+1): IMAD.HI, PRMT, LOP3, LDS, SHF per
//    probe against IMAD, LOP3, SHF, LOP3, LDS, SHF, SHF with the top bits of
//    one multiplicative hash, at the same or fewer false candidates
//    (host-simulated on the bench sets: k=1,000 4.04% vs 4.10% of words, k=10,000
//    9.7% vs 9.8%, DPI two-bit 4.3% vs 4.5%);
//  * byte layout (small gram sets): byte (cur * K ^ prev's top byte) >> 16.
constexpr uint32_t kP8HashMul = 0x9E3779B1u;
__host__ __device__ __forceinline__ uint32_t p8_mulhi(uint32_t x) {
#ifdef __CUDA_ARCH__
  return __umulhi(x, kP8HashMul);
#else
  return (uint32_t)(((unsigned long long)x * kP8HashMul) >> 32);
#endif
}
// byte offset of the (prev, cur) gram's 32-bit word in the 64 KB bit table
__host__ __device__ __forceinline__ uint32_t p8_word_off(uint32_t prev, uint32_t cur) {
#ifdef __CUDA_ARCH__
  const uint32_t pb = __byte_perm(prev, 0u, 0x4434);  // prev's top byte at bits 8..15
#else
  const uint32_t pb = (prev >> 16) & 0xFF00u;
#endif
  return (p8_mulhi(cur) ^ pb) & (kP8DmaskBytes - 4);
}
// funnel-shift amounts (low 5 bits used) of the gram's bit(s) in that word
__host__ __device__ __forceinline__ uint32_t p8_bit1(uint32_t cur) { return cur; }
__host__ __device__ __forceinline__ uint32_t p8_bit2(uint32_t cur) { return cur >> 8; }
#ifndef GLOP_P8_BIT2_PRMT
#define GLOP_P8_BIT2_PRMT 1
#endif
// two-bit layout, GLOP_P8_BIT2_PRMT: one PRMT puts cur's byte 1 at bits 0..7
// and prev's top byte at bits 8..15 (bits 16..31 are masked off); XORed into
// the word offset it also supplies the second bit's funnel amount, the same
// (cur >> 8) & 31 as p8_bit2, without the shift
__host__ __device__ __forceinline__ uint32_t p8_pb2(uint32_t prev, uint32_t cur) {
#ifdef __CUDA_ARCH__
  return __byte_perm(prev, cur, 0x4435);
#else
  return ((cur >> 8) & 0xFFu) | ((prev >> 16) & 0xFF00u) | ((cur & 0xFFu) * 0x01010000u);
#endif
}
__host__ __device__ __forceinline__ uint32_t p8_word_off2(uint32_t prev, uint32_t cur) {
  return (p8_mulhi(cur) ^ p8_pb2(prev, cur)) & (kP8DmaskBytes - 4);
}
// the gram's byte in the 64 KB d-mask table (byte layout)
__host__ __device__ __forceinline__ uint32_t p8_byte_off(uint32_t prev, uint32_t cur) {
  return ((cur * kP8HashMul) ^ (prev & 0xFF000000u)) >> (32 - kP8DmaskLog2);
}
// Above kP8Bits2Grams grams (DPI: ~39K) one bit per gram passes ~7% of the
// words on false positives alone; the "two bits in one word" layout (a
// blocked Bloom filter: bits p8_bit1 and p8_bit2 of the word) passes ~1%
// for two more instructions and no extra shared-memory wavefront per probe.
constexpr uint32_t kP8Bits2Grams = 12000;
// Small gram sets (kP8LaneGrams): the "lane-replicated" layout -- 512 words
// of 32 bits (16K one-bit buckets), each word stored once per bank, lane l's
// copy in bank l (byte offset w * 128 + 4 l).  Every lane reads only its own
// bank, so a probe instruction is ONE shared-memory wavefront instead of ~3.5
// for 32 random banks: the level-1 probes were ~55% of the kernel's
// wavefronts, and the LSU data pipe is what bounds it.  16K buckets keep the
// false candidates at a few percent up to ~1,000 grams (measured, 8 GB
// syslog: k=20 1.89 -> 1.73 ms, k=100 2.01 -> 1.79 ms, k=200 2.03 -> 1.92 ms;
// k=300 (1,188 grams) 2.03 -> 2.11 ms, so the one-bit layout keeps those).
// (below kP8LaneMinGrams the 64K-bucket byte layout's near-empty table lets
// most tiles skip the candidate stage entirely, which wins)
constexpr uint32_t kP8LaneGrams = 1000, kP8LaneMinGrams = 64;
__host__ __device__ __forceinline__ uint32_t p8_lane_off(uint32_t prev, uint32_t cur) {
#ifdef __CUDA_ARCH__
  const uint32_t pb = __byte_perm(prev, 0u, 0x4434);
#else
  const uint32_t pb = (prev >> 16) & 0xFF00u;
#endif
  return (p8_mulhi(cur) ^ pb) & (kP8DmaskBytes - 128u);  // word w at bits 7..15: w * 128
}
template <bool kBits, bool kTwo = false, bool kLane = false>
__device__ __forceinline__ uint32_t p8_dmask(const uint8_t* dm, uint32_t prev, uint32_t cur) {
  if (kLane) {  // dm = this lane's bank column
    const uint32_t w = *reinterpret_cast<const uint32_t*>(dm + p8_lane_off(prev, cur));
    return __funnelshift_r(w, w, p8_bit1(cur));
  }
  if (kBits) {  // bit p8_bit1 of the word, in bit 0 (bits 1..31: don't care)
    if (kTwo && GLOP_P8_BIT2_PRMT) {
      const uint32_t pb = p8_pb2(prev, cur);
      const uint32_t w = *reinterpret_cast<const uint32_t*>(dm + ((p8_mulhi(cur) ^ pb) & (kP8DmaskBytes - 4)));
      return __funnelshift_r(w, w, p8_bit1(cur)) & __funnelshift_r(w, w, pb);
    }
    const uint32_t w = *reinterpret_cast<const uint32_t*>(dm + p8_word_off(prev, cur));
    if (kTwo) return __funnelshift_r(w, w, p8_bit1(cur)) & __funnelshift_r(w, w, p8_bit2(cur));
    return __funnelshift_r(w, w, p8_bit1(cur));
  }
  return dm[p8_byte_off(prev, cur)];
}

// 1-D TMA bulk copy of aligned text A[lo, lo + kP8Stage) (clipped to the
// valid range [a, a + n)) into dst; bytes outside 16-byte granules are copied
// by the issuing lane.  One arrival (with tx bytes) on bar.
__device__ __forceinline__ void p8_issue(uint8_t* dst, uint32_t dst_a, uint32_t bar_a, const uint8_t* A, uint32_t a,
                                         unsigned long long n, unsigned long long lo) {
  const unsigned long long hi = lo + kP8Stage;
  if (lo >= a && hi <= a + n) {  // interior: one copy
    mbar_arrive_tx_a(bar_a, kP8Stage);
    bulk_g2s_a(dst_a, A + lo, kP8Stage, bar_a);
    return;
  }
  const unsigned long long vlo = lo > a ? lo : a, vhi = hi < a + n ? hi : a + n;
  unsigned long long tlo = (vlo + 15) & ~15ull, thi = vhi & ~15ull;
  if (thi < tlo) thi = tlo;
  for (unsigned long long x = vlo; x < tlo && x < vhi; ++x) dst[x - lo] = A[x];
  for (unsigned long long x = thi > vlo ? thi : vlo; x < vhi; ++x) dst[x - lo] = A[x];
  if (thi > tlo) {
    mbar_arrive_tx_a(bar_a, (uint32_t)(thi - tlo));
    bulk_g2s_a(dst_a + (uint32_t)(tlo - lo), A + tlo, (uint32_t)(thi - tlo), bar_a);
  } else {
    mbar_arrive_a(bar_a);
  }
}

// Sorts the warp's nb buffered hit keys (text offset << 24 | pattern id)
// and writes them as hits to dst (nullptr: the warp's staging region is full;
// the host grows it and reruns).  nb > kP8Hits means keys were dropped: the
// scan is flagged for the exact global-key fallback.  Whole warp.
// (inlined: as a real call it cost 5% at k=1,000 and 6% on the DPI set)
__device__ __forceinline__ uint32_t p8_flush(unsigned long long* hk, uint32_t nb, uint32_t lane, DevHit* dst,
                                          const uint32_t* pid_len, unsigned long long* g_count) {
  if (nb > kP8Hits) {
    if (lane == 0) {
      atomicAdd(g_count, (unsigned long long)nb);
      atomicOr(reinterpret_cast<unsigned int*>(g_count + 1), 1u);
    }
    return 0;
  }
  // batches are usually already in text order (a lane emits its candidates
  // in ascending offset, rounds and tiles ascend): sort only when needed
  if (!__all_sync(0xffffffffu, lane + 1 >= nb || hk[lane] < hk[lane + 1])) warp_sort_keys(hk, nb, lane);
  if (dst)
    for (uint32_t h = lane; h < nb; h += 32) {
      const unsigned long long key = hk[h];
      DevHit out;
      out.offset = key >> 24;
      out.pid = (uint32_t)key & 0xFFFFFFu;
      out.len = pid_len ? __ldg(pid_len + out.pid) : 8u;  // nullptr: every output at depth 8
      dst[h] = out;
    }
  __syncwarp();
  return nb;
}

// kL1: 5 = 3 for automata whose jump entries carry id lists (kOutList);
// 4 lane-replicated one-bit buckets (small gram sets);
// 0 byte d-mask buckets; 1 one-bit buckets; 2 one-bit buckets and a
// second level-2 bitmap probe (prefix_bit2_32) for large prefix sets; 3 as 2
// with two bits per gram in the level-1 word (kP8Bits2Grams).
// kCareful: a replayed lane always starts with an empty hit buffer.  Without
// it a replayed lane may start with up to GLOP_P8_FLUSH_AT keys, which is
// exact but sends a lane emitting more than kP8Hits - GLOP_P8_FLUSH_AT ids to
// the global-key fallback; the host picks kCareful for automata where one
// lane can emit that many (glop_trie_upload: p8_lane_emits), because its
// extra flush site costs ~3.5% of the k=1,000 scan (measured: 2.29 -> 2.37 ms).
template <bool kWalk, int kL1, typename Entry, bool kCareful>
__global__ void __launch_bounds__(kP8Threads, 1)
    pfac8_kernel(const DevTrie tr, const P8Params p, const P8Layout L) {
  using ET = EntryTraits<Entry>;
  constexpr bool kBits = kL1 != 0, kB2 = kL1 == 2 || kL1 == 3 || kL1 == 5, kTwo = kL1 == 3 || kL1 == 5,
                 kLane = kL1 == 4, kList2 = kL1 == 5;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint8_t* s_dmask = smem + L.dmask;
  const uint8_t* s_dm = kLane ? s_dmask + 4 * (threadIdx.x & 31) : s_dmask;  // (kLane: this lane's bank)
  const uint32_t* s_bm2 = reinterpret_cast<const uint32_t*>(smem + L.bm2);
  const uint32_t bm2_a = smem_u32(s_bm2);
  const uint8_t* s_cls = smem + L.cls;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars) + warp * 2;
  uint8_t* bufs = smem + L.bufs + (size_t)warp * 2 * kP8Stage;
  const uint32_t bufs_a = smem_u32(bufs), bars_a = smem_u32(bars);  // shared-window addresses
  uint16_t* q = reinterpret_cast<uint16_t*>(smem + L.queue) + warp * kP8Queue;
  unsigned long long* hk = reinterpret_cast<unsigned long long*>(smem + L.hits) + warp * kP8Hits;
  uint32_t* s_nh = reinterpret_cast<uint32_t*>(smem + L.nh) + warp;

  if (p.zero)  // (read only by kernels launched after this one)
    for (uint32_t i = blockIdx.x * kP8Threads + tid; i < p.nzero; i += gridDim.x * kP8Threads) p.zero[i] = 0;
  {
    const uint4* s = reinterpret_cast<const uint4*>(p.dmask8);
    uint4* d = reinterpret_cast<uint4*>(smem + L.dmask);
    for (uint32_t i = tid; i < kP8DmaskBytes / 16; i += kP8Threads) d[i] = s[i];
    s = reinterpret_cast<const uint4*>(tr.bm2_8);
    d = reinterpret_cast<uint4*>(smem + L.bm2);
    for (uint32_t i = tid; i < kP8Bm2Bytes / 16; i += kP8Threads) d[i] = s[i];
    if (kWalk && tid < 16) reinterpret_cast<uint4*>(smem + L.cls)[tid] = reinterpret_cast<const uint4*>(tr.cls)[tid];
    if (lane < 2) mbar_init(&bars[lane], 1);
    if (lane == 0) *s_nh = 0;
    if (tid == 0) fence_mbar_init();
  }
  __syncthreads();
  // this warp's contiguous segment of tiles [t0, t1)
  const uint32_t cta_lo = min(blockIdx.x * p.per, p.num_tiles), cta_hi = min(cta_lo + p.per, p.num_tiles);
  const uint32_t t0 = min(cta_lo + warp * p.sub, cta_hi), t1 = min(t0 + p.sub, cta_hi);
  const uint32_t a = (uint32_t)((uintptr_t)p.text & 15);
  const uint8_t* A = p.text - a;
  auto l2_prefetch = [&](uint32_t tt) {  // whole interior tiles only
    const unsigned long long lo = (unsigned long long)tt * kP8Tile;
    if (tt < t1 && lo >= a && lo + kP8Stage <= a + p.n) bulk_prefetch_l2(A + lo, kP8Stage);
  };
  if (lane == 0) {
    for (uint32_t b = 0; b < 2; ++b)
      if (t0 + b < t1)
        p8_issue(bufs + b * kP8Stage, bufs_a + b * kP8Stage, bars_a + 8 * b, A, a, p.n,
                 (unsigned long long)(t0 + b) * kP8Tile);
    for (uint32_t b = 0; b < kP8L2Pf; ++b) l2_prefetch(t0 + 2 + b);
  }
  const unsigned long long own_end = p.own + a, n_end = p.n + a;  // aligned coordinates
  // interior tiles: t >= 1, all kP8Tile starts owned, the whole stage inside
  // the text -- no range masks
  const uint32_t t_int_hi =
      n_end < kP8Stage ? 0u : (uint32_t)min(own_end / kP8Tile, (n_end - kP8Stage) / kP8Tile + 1);
  const uint32_t gw = blockIdx.x * kP8Warps + warp;
  DevHit* region = p.staging + (unsigned long long)gw * p.region;
  uint32_t cursor = 0;  // hits written to this warp's region
  uint32_t ltmask;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(ltmask));

  auto flush = [&](uint32_t nb) {
    const bool fits = cursor + nb <= p.region;
    cursor += p8_flush(hk, nb, lane, fits ? region + cursor : nullptr, kWalk ? tr.pid_len : nullptr, p.g_count);
    if (lane == 0) *s_nh = 0;
    __syncwarp();
  };

  // text offset of the window's byte 0, carried across tiles
  unsigned long long off0 = p.base + (unsigned long long)t0 * kP8Tile - a;
  // A tile's last, partial drain round is carried into the next tile's first
  // round (kCarry): its candidates' words, offset mask, word index and window
  // offset stay in registers, so the few candidates of small rule sets share
  // rounds across tiles (k=10: 1.63 -> 1.57 ms).  Only the byte layout (small
  // gram sets): with the other layouts' ~20 candidates per tile the extra
  // live registers cost more than the saved rounds (k=1,000 2.20 -> 2.31 ms,
  // k=100 1.76 -> 1.84 ms).  Not for kWalk automata: their deeper walk reads
  // the tile's shared-memory window.
  constexpr bool kCarry = !kWalk && kL1 == 0 && GLOP_P8_CARRY;
  uint32_t cw0 = 0, cw1 = 0, cw2 = 0, cmm = 0, ci = 1, cL = 0;  // cL: carried lanes (warp-uniform)
  unsigned long long cbase = 0;
  for (uint32_t t = t0, k = 0; t < t1; ++t, ++k, off0 += kP8Tile) {
    const uint32_t b = k & 1;
    mbar_wait_a(bars_a + 8 * b, (k >> 1) & 1);
    const uint8_t* sb = bufs + b * kP8Stage;
    const uint32_t* sw = reinterpret_cast<const uint32_t*>(sb);
    const bool edge = t == 0 || t >= t_int_hi;
    uint32_t lo = 0, s_hi = kP8Tile, avail = kP8Stage;
    if (edge) {
      const unsigned long long tA = (unsigned long long)t * kP8Tile;
      s_hi = (uint32_t)min(own_end - tA, (unsigned long long)kP8Tile);
      avail = (uint32_t)min(n_end - tA, 0x7FFFFFFFull);
      lo = t == 0 ? a : 0;
    }

    unsigned long long ebase = off0;  // window offset of the candidate being checked (carried: its own tile's)
    auto emit = [&](uint32_t c, uint32_t pid) {
      const unsigned long long key = ((ebase + c) << 24) | pid;
      if (p.mode == 0) {
        const uint32_t slot = atomicAdd(s_nh, 1u);
        if (slot < kP8Hits) hk[slot] = key;
      } else {
        const unsigned long long slot = atomicAdd(p.g_count + 3, 1ull);
        if (slot < p.keys_cap) p.keys[slot] = key;
      }
    };
    auto emit_state = [&](uint32_t c, uint32_t st) {
      for (uint32_t o = __ldg(tr.out_off + st), oe = __ldg(tr.out_off + st + 1); o < oe; ++o)
        emit(c, __ldg(tr.out_pid + o));
    };
    // exact check of candidate start c (window byte) with 8-byte key (lo32, hi32)
    auto exact = [&](uint32_t c, uint32_t klo, uint32_t khi) {
      const unsigned long long key = (unsigned long long)klo | ((unsigned long long)khi << 32);
      const uint32_t cap_log2 = tr.jump_cap_log2, hmask = (1u << cap_log2) - 1;
      for (uint32_t h = jump_slot(key, cap_log2);; h = (h + 1) & hmask) {
        const JumpEntry e = tr.jump[h];
        if (!e.state1) return;
        if (e.key != key) continue;
        uint32_t st = e.state1 - 1;
        if (e.out != kOutNone) {
          if (e.out < kOutList) emit(c, e.out);
          else if (e.out == kOutMany) emit_state(c, st);
          else if constexpr (kList2) {
            // rule sets with shared prefixes (DPI): the first two ids loaded
            // together, one L2 round trip (DPI 1.75 -> 1.70 ms; the same code
            // in every instantiation cost k=1,000 2.8% and k=10,000 1.9%)
            const uint32_t o = e.out & 0xFFFFFFu, nn = ((e.out >> 24) & 0x7Fu) + 1;
            const uint32_t v0 = __ldg(tr.out_pid + o), v1 = __ldg(tr.out_pid + o + 1);
            const uint32_t v2 = nn > 2 ? __ldg(tr.out_pid + o + 2) : 0u;
            if (p.mode == 0) {  // the list's slots in one shared-memory atomic
              const unsigned long long kb = (ebase + c) << 24;
              const uint32_t slot = atomicAdd(s_nh, nn);
              if (slot < kP8Hits) hk[slot] = kb | v0;
              if (slot + 1 < kP8Hits) hk[slot + 1] = kb | v1;
              if (nn > 2 && slot + 2 < kP8Hits) hk[slot + 2] = kb | v2;
              for (uint32_t k2 = 3; k2 < nn; ++k2)
                if (slot + k2 < kP8Hits) hk[slot + k2] = kb | __ldg(tr.out_pid + o + k2);
            } else {
              emit(c, v0);
              emit(c, v1);
              if (nn > 2) emit(c, v2);
              for (uint32_t k2 = 3; k2 < nn; ++k2) emit(c, __ldg(tr.out_pid + o + k2));
            }
          } else {
            for (uint32_t o = e.out & 0xFFFFFFu, oe = o + ((e.out >> 24) & 0x7Fu) + 1; o < oe; ++o)
              emit(c, __ldg(tr.out_pid + o));
          }
        }
        if (kWalk && tr.lmax > 8) {  // deeper levels: scan.hpp:142-168
          const unsigned long long tA = (unsigned long long)t * kP8Tile;
          const uint32_t av = (uint32_t)min(n_end - tA, 0x7FFFFFFFull);
          const Entry* T = reinterpret_cast<const Entry*>(tr.table);
          for (uint32_t j = c + 8; j < av; ++j) {
            const uint32_t byte = j < kP8Stage ? sb[j] : __ldg(p.text + (tA + j - a));
            const uint32_t x = __ldg(T + st * tr.C + s_cls[byte]);
            if (!x) break;
            st = x & ET::kMask;
            if (x & ET::kFlag) emit_state(c, st);
          }
        }
        return;
      }
    };

    // Level 1 over the whole tile in one pass: lane l samples tile words
    // 8 l + 1 .. 8 l + 8 (first half) and 256 + 8 l + 1 .. 256 + 8 l + 8 (second
    // half), which covers candidates 0..kP8Tile-1.  Candidate words enter the
    // queue q (u16: word << 4 | d-mask) in text order -- one packed shuffle
    // scan gives both halves' prefixes -- and are checked 32 per round.
    uint32_t qt = 0;
    {
      // quarter k of the tile samples words 128 k + 1 .. 128 k + 128; lane l
      // takes words 128 k + 4 l + 1 .. + 4 from one conflict-free LDS.128
      // (consecutive lanes, consecutive 16 B) and the next lane's first word
      uint32_t mq[4], mm4[4][4];
#pragma unroll
      for (uint32_t hf = 0; hf < 2; ++hf) {
        const uint32_t W = hf * (kP8Tile / 8);
        const uint4 va = reinterpret_cast<const uint4*>(sw + W)[lane];
        const uint4 vb = reinterpret_cast<const uint4*>(sw + W)[32 + lane];
        const uint32_t wn = sw[W + kP8Tile / 8];
        const uint32_t na = __shfl_sync(0xffffffffu, lane == 0 ? vb.x : va.x, (lane + 1) & 31);
        uint32_t nb = __shfl_down_sync(0xffffffffu, vb.x, 1);
        if (lane == 31) nb = wn;
        uint32_t* a = mm4[2 * hf];
        uint32_t* b = mm4[2 * hf + 1];
        a[0] = p8_dmask<kBits, kTwo, kLane>(s_dm, va.x, va.y);
        a[1] = p8_dmask<kBits, kTwo, kLane>(s_dm, va.y, va.z);
        a[2] = p8_dmask<kBits, kTwo, kLane>(s_dm, va.z, va.w);
        a[3] = p8_dmask<kBits, kTwo, kLane>(s_dm, va.w, na);
        b[0] = p8_dmask<kBits, kTwo, kLane>(s_dm, vb.x, vb.y);
        b[1] = p8_dmask<kBits, kTwo, kLane>(s_dm, vb.y, vb.z);
        b[2] = p8_dmask<kBits, kTwo, kLane>(s_dm, vb.z, vb.w);
        b[3] = p8_dmask<kBits, kTwo, kLane>(s_dm, vb.w, nb);
        if (kBits) {  // byte j = probe j's bit 0
          mq[2 * hf] = __byte_perm(__byte_perm(a[0], a[1], 0x40), __byte_perm(a[2], a[3], 0x40), 0x5410) & 0x01010101u;
          mq[2 * hf + 1] = __byte_perm(__byte_perm(b[0], b[1], 0x40), __byte_perm(b[2], b[3], 0x40), 0x5410) & 0x01010101u;
        } else {
          mq[2 * hf] = __byte_perm(a[0] | (a[1] << 8), a[2] | (a[3] << 8), 0x5410);
          mq[2 * hf + 1] = __byte_perm(b[0] | (b[1] << 8), b[2] | (b[3] << 8), 0x5410);
        }
      }
      if (__ballot_sync(0xffffffffu, (mq[0] | mq[1] | mq[2] | mq[3]) != 0)) {
        // candidate words per quarter (d-masks are < 16: adding 0x7F to a
        // byte sets its top bit iff the byte is non-zero; bit layout: bytes
        // are 0/1), packed 8 bits per quarter (<= 128 each): one shuffle scan
        // gives all four prefixes
        auto nz = [](uint32_t x) { return kBits ? __popc(x) : __popc((x + 0x7F7F7F7Fu) & 0x80808080u); };
        const uint32_t cnt = nz(mq[0]) | (nz(mq[1]) << 8) | (nz(mq[2]) << 16) | (nz(mq[3]) << 24);
        uint32_t incl = cnt;
#pragma unroll
        for (uint32_t o = 1; o < 32; o <<= 1)  // the shuffle's own in-range predicate guards the add
          asm volatile(
              "{\n\t.reg .pred p;\n\t.reg .b32 x;\n\t"
              "shfl.sync.up.b32 x|p, %0, %1, 0, 0xffffffff;\n\t"
              "@p add.u32 %0, %0, x;\n}"
              : "+r"(incl)
              : "r"(o));
        const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t ex = incl - cnt;
        // 16 predicated u16 stores through a running shared-memory address
        // per quarter (value = word << 4 | d-mask; the word base is per lane)
        uint32_t vl;  // opaque, so each value is one IADD3 (vl + m + const)
        asm("mov.u32 %0, %1;" : "=r"(vl) : "r"((4 * lane + 1) << 4));
        uint32_t base = smem_u32(q);
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) {
          uint32_t qa = base + 2 * ((ex >> (8 * k)) & 0xFFu);
#pragma unroll
          for (uint32_t j = 0; j < 4; ++j) {
            if (kBits ? (mq[k] & (1u << (8 * j))) != 0 : mm4[k][j] != 0) {
              const uint32_t m = kBits ? 1u : mm4[k][j];
              asm volatile("st.shared.u16 [%0], %1;" ::"r"(qa), "r"(vl + ((128 * k + j) << 4) + m) : "memory");
              qa += 2;
            }
          }
          base += 2 * ((tot >> (8 * k)) & 0xFFu);
        }
        qt = (tot & 0xFFu) + ((tot >> 8) & 0xFFu) + ((tot >> 16) & 0xFFu) + (tot >> 24);
        __syncwarp();
      }
    }
    {
      // rounds over the virtual list [carried lanes (cL), this tile's queue (qt)]
      const uint32_t total = (kCarry ? cL : 0u) + qt;
      if (kCarry) cL = 0;
#pragma unroll 1
      for (uint32_t qh = 0; qh < total; qh += 32) {
        const uint32_t pend = total - qh;
        // ---- 8-byte keys of up to 32 candidate words -> prefix bitmap
        const uint32_t v = qh + lane, ncar = kCarry ? total - qt : 0u;
        uint32_t i, mm, w0, w1, w2;
        if (kCarry && v < ncar) {  // carried from an earlier tile (first round only)
          i = ci, mm = cmm, w0 = cw0, w1 = cw1, w2 = cw2;
          ebase = cbase;
        } else {
          const uint32_t e = v < total ? q[v - ncar] : 16u;  // idle lanes: word 1, no bits
          i = e >> 4;
          mm = kBits ? (e & 1u) * 15u : e & 15u;  // bit layout: all four offsets
          w0 = sw[i - 1], w1 = sw[i], w2 = sw[i + 1];
          ebase = off0;
          if (edge) {
#pragma unroll
            for (uint32_t d = 1; d <= 4; ++d) {
              const uint32_t c = 4 * i - d;
              if (c < lo || c >= s_hi || c + 8 > avail) mm &= ~(1u << (d - 1));
            }
          }
        }
        if (kCarry && pend < 32 && t + 1 < t1) {  // partial round: carry it into the next tile
          cw0 = w0, cw1 = w1, cw2 = w2, cmm = lane < pend ? mm : 0u, ci = i, cbase = ebase;
          cL = pend;
          break;
        }
        uint32_t surv = 0;
#pragma unroll
        for (uint32_t d = 1; d <= 4; ++d) {
          const uint32_t x = prefix_hash32(__funnelshift_r(w0, w1, 32 - 8 * d), __funnelshift_r(w1, w2, 32 - 8 * d));
          // probe only for the d-mask's offsets: predicated-off lanes take no
          // shared-memory bank slot (fewer conflicts)
          uint32_t word = x;
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t@p ld.shared.b32 %0, [%1];\n}"
                       : "+r"(word)
                       : "r"(bm2_a + ((x >> (32 - kP8Bm2Log2 + 5)) << 2)), "r"(mm & (1u << (d - 1))));
          // rotate bit (x >> 14) & 31 of the bitmap word to position d - 1
          surv |= __funnelshift_r(word, word, (x >> (32 - kP8Bm2Log2)) + (33 - d)) & (1u << (d - 1));
          if (kB2) {  // second, independent 18-bit slice of the same key hash
            const uint32_t x2 = prefix_hash2(x);
            uint32_t word2 = x2;
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t@p ld.shared.b32 %0, [%1];\n}"
                         : "+r"(word2)
                         : "r"(bm2_a + ((x2 >> (32 - kP8Bm2Log2 + 5)) << 2)), "r"(surv & (1u << (d - 1))));
            surv &= ~(1u << (d - 1)) | __funnelshift_r(word2, word2, (x2 >> (32 - kP8Bm2Log2)) + (33 - d));
          }
        }
        surv &= mm;
        const uint32_t runmask = __ballot_sync(0xffffffffu, surv != 0);
        if (!runmask) continue;
        // ---- exact check of the survivors; a pass that overflows the hit
        // buffer is dropped and replayed lane by lane (lanes hold ascending
        // candidates), flushing in between
        auto run_lanes = [&](uint32_t mask) {
          if ((mask >> lane) & 1u) {
            uint32_t sv = surv;
            while (sv) {
              const uint32_t d = 32 - __clz(sv);  // 4..1: ascending candidate offsets
              sv &= ~(1u << (d - 1));
              const uint32_t sh = 32 - 8 * d;
              exact(4 * i - d, __funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh));
            }
          }
          __syncwarp();
          const uint32_t nb = *s_nh;
          __syncwarp();
          return nb;
        };
        const uint32_t nb0 = *s_nh;  // <= GLOP_P8_FLUSH_AT
        if constexpr (kCareful) {
          const uint32_t nb = run_lanes(runmask);
          if (p.mode == 0) {
            if (nb > kP8Hits) {
              // replay: flush the earlier rounds' keys, then run each lane
              // alone and flush after it
              if (lane == 0) *s_nh = nb0;
              __syncwarp();
              if (nb0) flush(nb0);
#pragma unroll 1
              for (uint32_t redo = runmask; redo; redo &= redo - 1) {
                const uint32_t nl = run_lanes(redo & (0u - redo));
                if (nl) flush(nl);
              }
            } else if (nb > GLOP_P8_FLUSH_AT) {
              flush(nb);
            }
          }
        } else {
          uint32_t mask = runmask, redo = 0;
          bool first = true;
          for (;;) {
            const uint32_t nb = run_lanes(mask);
            if (p.mode == 0) {
              if (first && nb > kP8Hits) {  // replay lane by lane from the earlier rounds' keys
                if (lane == 0) *s_nh = nb0;
                __syncwarp();
                redo = runmask;
              } else if (nb > GLOP_P8_FLUSH_AT) {
                flush(nb);
              }
            }
            first = false;
            if (!redo) break;
            mask = redo & (0u - redo);
            redo &= redo - 1;
          }
        }
      }
    }
    // buffer b is free: refill it with the segment's tile t + 2 (interior
    // tiles, the common case, with one 32-bit test: the general p8_issue
    // cost ~35 warp instructions per tile in 64-bit range checks)
    __syncwarp();
    if (t + 2 < t1) {
      if (GLOP_P8_FASTREFILL && t + 2 < t_int_hi) {
        if (lane == 0) {
          fence_proxy_async();
          mbar_arrive_tx_a(bars_a + 8 * b, kP8Stage);
          bulk_g2s_a(bufs_a + b * kP8Stage, A + (size_t)(t + 2) * kP8Tile, kP8Stage, bars_a + 8 * b);
        }
      } else if (lane == 0) {
        fence_proxy_async();
        p8_issue(bufs + b * kP8Stage, bufs_a + b * kP8Stage, bars_a + 8 * b, A, a, p.n,
                 (unsigned long long)(t + 2) * kP8Tile);
      }
      if (kP8L2Pf && lane == 0) l2_prefetch(t + 2 + kP8L2Pf);
    }
  }
  if (p.mode == 0) {
    __syncwarp();
    const uint32_t nb = *s_nh;
    __syncwarp();
    if (nb) flush(nb);
    if (lane == 0) {
      p.counts[gw] = cursor;
      if (cursor) {
        atomicAdd(p.g_count, (unsigned long long)cursor);
        atomicMax(p.g_count + 2, (unsigned long long)cursor);
      }
    }
  }
}

// sum over i in [0, n) of min(counts[i], cap), in every thread of the CTA
// (s_red: 32 words of shared memory; blockDim.x a multiple of 32)
__device__ __forceinline__ unsigned long long block_sum_counts(const unsigned long long* counts, uint32_t n,
                                                               unsigned long long cap, unsigned long long* s_red) {
  unsigned long long s = 0;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) s += min(counts[i], cap);
  for (uint32_t o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();  // (s_red may still be read from a previous call)
  if (lane == 0) s_red[w] = s;
  __syncthreads();
  s = lane < blockDim.x / 32 ? s_red[lane] : 0ull;
  for (uint32_t o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// Exclusive prefix of min(counts[g0 + j], cap) over j in [0, n] into
// s_pre[0..n] (n <= kRangeMax), computed by warp 0 32 entries at a time;
// the caller synchronizes the CTA before reading it.
constexpr uint32_t kRangeMax = 64;
__device__ __forceinline__ void range_prefix(const unsigned long long* counts, uint32_t g0, uint32_t n,
                                             unsigned long long cap, unsigned long long* s_pre) {
  if (threadIdx.x >= 32) return;
  const uint32_t lane = threadIdx.x;
  unsigned long long run = 0;
  for (uint32_t j0 = 0; j0 < n; j0 += 32) {
    const uint32_t j = j0 + lane;
    const unsigned long long c = j < n ? min(counts[g0 + j], cap) : 0ull;
    unsigned long long incl = c;
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (j < n) s_pre[j] = run + incl - c;
    run += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) s_pre[n] = run;
}

// Concatenates the per-warp regions (each already in text order) in warp
// order, each CTA a contiguous range of regions: the range's output offset is
// the sum of the counts before it (computed here -- no separate prefix
// launch), the regions' offsets inside the range a prefix in shared memory,
// and each warp copies whole regions (round robin), so the regions' count
// loads and copies overlap instead of running one region after another.
// Launched before the host has looked at the scan's flags: records past
// `cap` or beyond a region are not copied, and a flagged scan is redone.
template <typename Rec>
__global__ void __launch_bounds__(256) gather_regions_kernel(const unsigned long long* counts, uint32_t regions,
                                                             unsigned long long region, const Rec* staging,
                                                             Rec* out, unsigned long long cap) {
  __shared__ unsigned long long s_red[32], s_pre[kRangeMax + 1];
  const uint32_t per = (regions + gridDim.x - 1) / gridDim.x;
  const uint32_t g0 = min(blockIdx.x * per, regions), g1 = min(g0 + per, regions);
  const unsigned long long base = block_sum_counts(counts, g0, region, s_red);
  if (per > kRangeMax) {  // (not with the launch geometries used; kept exact)
    unsigned long long dst = base;
    for (uint32_t g = g0; g < g1; ++g) {
      const unsigned long long c = min(counts[g], region);
      const Rec* src = staging + (unsigned long long)g * region;
      for (unsigned long long h = threadIdx.x; h < c && dst + h < cap; h += blockDim.x) out[dst + h] = src[h];
      dst += c;
    }
    return;
  }
  range_prefix(counts, g0, g1 - g0, region, s_pre);
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (uint32_t j = threadIdx.x >> 5; j < g1 - g0; j += nw) {
    const unsigned long long d0 = base + s_pre[j], c = s_pre[j + 1] - s_pre[j];
    const Rec* src = staging + (unsigned long long)(g0 + j) * region;
    for (unsigned long long h = lane; h < c && d0 + h < cap; h += 32) out[d0 + h] = src[h];
  }
}

}  // namespace glop
