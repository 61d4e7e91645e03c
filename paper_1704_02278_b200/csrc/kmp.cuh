// kmp.cuh -- K4: chunk-parallel KMP (kmp_search, kmp.hpp:41-69) with the
// reference's exact comparison count.
//
// The reference's failure-function loop is replayed on the host into a DFA
// over (state, byte): entry = next state (13 bits) | match << 13 |
// comparisons << 14, so the sequential comparison count is reproduced step
// by step.  Each lane owns 144 consecutive match END positions (144 = 9 x 16
// bytes: the warp's LDS.128 hit distinct banks); the state at its first
// position is recovered by a warm-up over the previous m-1 bytes (the KMP
// state depends only on them).  In state 0 a byte other than p[0] costs one
// comparison and keeps state 0, so 16-byte groups without p[0] are skipped
// (SWAR test on the registers of one LDS.128) and inside a group the walk
// jumps to the next p[0]; only bytes after a p[0] walk the DFA.
//
// Work split as in pfac8.cuh: one 512-thread CTA per SM, each warp streams a
// CONTIGUOUS segment of 4,608-byte warp tiles through a private
// double-buffered TMA pipeline -- no CTA barriers.  A warp's matches come out
// in text order tile by tile (a tile's few keys are warp-sorted in shared
// memory), so the output is the concatenation of the per-warp staging
// regions (gather_regions_kernel).  A tile with more matches
// than the buffer flags the exact global-key fallback (CUB radix sort).
#pragma once
#include <type_traits>

#include "glop_kernels.cuh"
#include "pfac8.cuh"

namespace glop {

constexpr int kK3Warps = 16;
constexpr int kK3Threads = kK3Warps * 32;
constexpr uint32_t kK3Chunk = 144;                 // end positions per lane
constexpr uint32_t kK3Tile = kK3Chunk * 32;        // 4,608 per warp tile
constexpr uint32_t kK3Pre = 64;                    // warm-up bytes kept before the tile
constexpr uint32_t kK3Stage = kK3Pre + kK3Tile + 16;
constexpr uint32_t kK3Hits = 64;                   // match keys per warp tile in smem
constexpr uint32_t kK3SmemDfaMax = 48;             // patterns up to 48 bytes keep the DFA in smem

struct K3Layout {
  uint32_t bufs, bars, keys, nh, dfa, total;
};

__host__ __device__ inline K3Layout make_k3_layout(uint32_t m, bool smem_dfa) {
  K3Layout L;
  uint32_t o = 0;
  L.bufs = o; o += kK3Warps * 2 * kK3Stage;
  L.bars = o; o += kK3Warps * 2 * 8;
  L.keys = o; o += kK3Warps * kK3Hits * 8;
  L.nh = o; o += kK3Warps * 4;
  L.dfa = align16(o); o = L.dfa + (smem_dfa ? m * 1024 : 0);
  L.total = o;
  return L;
}

struct K3Params {
  const uint8_t* text;
  unsigned long long n, own, end_lim, base;  // starts < own; ends (last byte of a match) < end_lim
  unsigned long long skip;                   // left context: starts and comparisons from position skip on
  uint32_t m, p0, num_tiles, per, sub;
  const uint32_t* dfa;                  // m x 256
  unsigned long long* staging;          // per-warp regions of start offsets
  unsigned long long region;
  unsigned long long* counts;           // matches per region
  unsigned long long* g_count;          // [0] total, [1] flags, [2] comparisons, [3] max region use
  unsigned long long* comparisons;
  int mode;                             // 0: per-warp ordered staging; 1: global keys (fallback)
  unsigned long long* keys;
  unsigned long long keys_cap;
};

// TMA window: dst[0, bytes) <- A[lo, lo + bytes) clipped to [a, a + n)
// (lo may be negative); partial 16-byte granules by the issuing thread.
__device__ __forceinline__ void k2_issue(uint8_t* dst, uint64_t* bar, const uint8_t* A, uint32_t a,
                                         unsigned long long n, long long lo, uint32_t bytes) {
  const long long hi = lo + bytes;
  if (lo >= (long long)a && hi <= (long long)(a + n)) {  // interior: one copy
    mbar_arrive_tx(bar, bytes);
    bulk_g2s(dst, A + lo, bytes, bar);
    return;
  }
  const long long vlo = lo > (long long)a ? lo : (long long)a;
  const long long vhi = hi < (long long)(a + n) ? hi : (long long)(a + n);
  long long tlo = (vlo + 15) & ~15ll, thi = vhi & ~15ll;
  if (thi < tlo) thi = tlo;
  for (long long x = vlo; x < tlo && x < vhi; ++x) dst[x - lo] = A[x];
  for (long long x = thi > vlo ? thi : vlo; x < vhi; ++x) dst[x - lo] = A[x];
  if (thi > tlo) {
    mbar_arrive_tx(bar, (uint32_t)(thi - tlo));
    bulk_g2s(dst + (tlo - lo), A + tlo, (uint32_t)(thi - tlo), bar);
  } else {
    mbar_arrive(bar);
  }
}

// bit 7 of byte k set where byte k of w may equal p0 (x4 = p0 * 0x01010101);
// exact for the first such byte, possibly spurious above it -- harmless:
// a DFA step in state 0 on a non-p0 byte is one comparison and stays in 0.
__device__ __forceinline__ uint32_t k2_zero_bytes(uint32_t w, uint32_t x4) {
  const uint32_t t = w ^ x4;
  return (t - 0x01010101u) & ~t & 0x80808080u;
}
// bits 7,15,23,31 -> bits 0..3
__device__ __forceinline__ uint32_t k2_gather4(uint32_t z) { return (((z >> 7) * 0x00204081u) >> 21) & 15u; }

template <bool kSmemDfa>
__global__ void __launch_bounds__(kK3Threads, 1) kmp3_kernel(const K3Params p, const K3Layout L) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars) + warp * 2;
  uint8_t* bufs = smem + L.bufs + (size_t)warp * 2 * kK3Stage;
  unsigned long long* hk = reinterpret_cast<unsigned long long*>(smem + L.keys) + warp * kK3Hits;
  uint32_t* s_nh = reinterpret_cast<uint32_t*>(smem + L.nh) + warp;
  uint32_t* s_dfa = reinterpret_cast<uint32_t*>(smem + L.dfa);
  if (kSmemDfa)
    for (uint32_t i = tid; i < p.m * 64; i += kK3Threads)
      reinterpret_cast<uint4*>(s_dfa)[i] = reinterpret_cast<const uint4*>(p.dfa)[i];
  if (lane < 2) mbar_init(&bars[lane], 1);
  if (lane == 0) *s_nh = 0;
  if (tid == 0) fence_mbar_init();
  __syncthreads();
  const uint32_t* D = kSmemDfa ? s_dfa : p.dfa;
  const uint32_t a = (uint32_t)((uintptr_t)p.text & 15);
  const uint8_t* A = p.text - a;                   // 16-aligned; text position x is A[x + a]
  const unsigned long long e_end = p.end_lim + a;  // end positions, A coordinates
  const unsigned long long o_end = p.own + a;      // comparisons counted for positions < own
  const uint32_t cta_lo = min(blockIdx.x * p.per, p.num_tiles), cta_hi = min(cta_lo + p.per, p.num_tiles);
  const uint32_t t0 = min(cta_lo + warp * p.sub, cta_hi), t1 = min(t0 + p.sub, cta_hi);
  if (lane == 0)
    for (uint32_t b = 0; b < 2; ++b)
      if (t0 + b < t1)
        k2_issue(bufs + b * kK3Stage, &bars[b], A, a, p.n, (long long)(t0 + b) * kK3Tile - kK3Pre, kK3Stage);
  const uint32_t x4 = p.p0 * 0x01010101u, m = p.m;
  const uint32_t gw = blockIdx.x * kK3Warps + warp;
  unsigned long long* region = p.staging + (unsigned long long)gw * p.region;
  unsigned long long cmp_total = 0;
  uint32_t cursor = 0;  // matches written to this warp's region

  for (uint32_t t = t0, k = 0; t < t1; ++t, ++k) {
    const uint32_t b = k & 1;
    mbar_wait(&bars[b], (k >> 1) & 1);
    const uint8_t* win = bufs + b * kK3Stage;  // window byte y holds A[tT - kK3Pre + y]
    const unsigned long long tT = (unsigned long long)t * kK3Tile;
    auto abyte = [&](unsigned long long x) -> uint32_t {  // A coordinate, a <= x < a + n
      const long long y = (long long)(x - tT) + kK3Pre;
      return (y >= 0 && y < (long long)kK3Stage) ? win[y] : __ldg(A + x);
    };
    auto record = [&](unsigned long long x) {  // match ending at A coordinate x
      if (x + 1 < a + p.skip + m) return;  // starts in the left context belong to the previous shard
      const unsigned long long start = p.base + x - a + 1 - m;
      if (p.mode == 0) {
        const uint32_t slot = atomicAdd(s_nh, 1u);
        if (slot < kK3Hits) hk[slot] = start;
      } else {
        const unsigned long long slot = atomicAdd(p.g_count, 1ull);
        if (slot < p.keys_cap) p.keys[slot] = start;
      }
    };
    // Walks window bytes [yf, yt) from state j; kCount: add the reference's
    // comparisons, kRecord: record matches (the warm-up does neither, a
    // shard's halo only records -- its comparisons belong to the next shard).
    auto walk = [&](auto kCount, auto kRecord, uint32_t yf, uint32_t yt, uint32_t& j, unsigned long long& cmp) {
      for (uint32_t g = yf & ~15u; g < yt; g += 16) {
        const uint32_t kb = yf > g ? yf - g : 0u;
        const uint32_t ke = min(yt - g, 16u);
        const uint4 v = *reinterpret_cast<const uint4*>(win + g);
        const uint32_t z0 = k2_zero_bytes(v.x, x4), z1 = k2_zero_bytes(v.y, x4), z2 = k2_zero_bytes(v.z, x4),
                       z3 = k2_zero_bytes(v.w, x4);
        if (j == 0 && !(z0 | z1 | z2 | z3)) {
          if (decltype(kCount)::value) cmp += ke - kb;
          continue;
        }
        uint32_t mask = k2_gather4(z0) | (k2_gather4(z1) << 4) | (k2_gather4(z2) << 8) | (k2_gather4(z3) << 12);
        mask &= (1u << ke) - 1u;
        uint32_t kk = kb;
        while (kk < ke) {
          if (j == 0) {
            const uint32_t mk = mask & (0xFFFFFFFFu << kk);
            if (!mk) {
              if (decltype(kCount)::value) cmp += ke - kk;
              break;
            }
            const uint32_t s = __ffs(mk) - 1;
            if (decltype(kCount)::value) cmp += s - kk;
            kk = s;
          }
          const uint32_t e = D[j * 256 + win[g + kk]];
          if (decltype(kCount)::value) cmp += e >> 14;
          if (decltype(kRecord)::value && (e & 0x2000u)) record(tT - kK3Pre + g + kk);
          j = e & 0x1FFFu;
          ++kk;
        }
      }
    };
    unsigned long long c0 = tT + (unsigned long long)lane * kK3Chunk;
    if (c0 < a + p.skip) c0 = a + p.skip;  // (left context: warm-up only)
    const unsigned long long c1 = min(tT + (unsigned long long)(lane + 1) * kK3Chunk, e_end);
    if (c0 < c1) {
      const uint32_t y0 = (uint32_t)(c0 - tT) + kK3Pre, y1 = (uint32_t)(c1 - tT) + kK3Pre;
      // warm-up: the state at c0 from the m-1 bytes before it (clamped to the text start)
      uint32_t j = 0;
      unsigned long long cmp = 0;
      const unsigned long long wlo = c0 - min(c0 - a, (unsigned long long)(m - 1));
      if (wlo + kK3Pre >= tT) {
        walk(std::false_type{}, std::false_type{}, (uint32_t)(wlo + kK3Pre - tT), y0, j, cmp);
      } else {  // long patterns: warm-up bytes before the window
        for (unsigned long long x = wlo; x < c0; ++x) {
          const uint32_t bt = abyte(x);
          if (j != 0 || bt == p.p0) j = D[j * 256 + bt] & 0x1FFFu;
        }
      }
      if (c1 <= o_end) {
        walk(std::true_type{}, std::true_type{}, y0, y1, j, cmp);
      } else {  // the chunk reaches into the shard's halo
        const uint32_t yo = c0 < o_end ? (uint32_t)(o_end - tT) + kK3Pre : y0;
        walk(std::true_type{}, std::true_type{}, y0, yo, j, cmp);
        walk(std::false_type{}, std::true_type{}, yo, y1, j, cmp);
      }
      cmp_total += cmp;
    }
    __syncwarp();
    // buffer b is free: refill it with the segment's tile t + 2
    if (lane == 0 && t + 2 < t1) {
      fence_proxy_async();
      k2_issue(bufs + b * kK3Stage, &bars[b], A, a, p.n, (long long)(t + 2) * kK3Tile - kK3Pre, kK3Stage);
    }
    if (p.mode == 0) {
      const uint32_t nb = *s_nh;
      if (nb) {  // this tile's matches, in order, appended to the region
        if (nb > kK3Hits) {
          if (lane == 0) atomicOr(reinterpret_cast<unsigned int*>(p.g_count + 1), 1u);
        } else {
          warp_sort_keys(hk, nb, lane);
          if (cursor + nb <= p.region)
            for (uint32_t h = lane; h < nb; h += 32) region[cursor + h] = hk[h];
        }
        cursor += nb;
        __syncwarp();
        if (lane == 0) *s_nh = 0;
        __syncwarp();
      }
    }
  }
  for (int o = 16; o; o >>= 1) cmp_total += __shfl_xor_sync(0xffffffffu, cmp_total, o);
  if (lane == 0) {
    if (cmp_total) atomicAdd(p.comparisons, cmp_total);
    if (p.mode == 0) {
      p.counts[gw] = cursor;
      if (cursor) {
        atomicAdd(p.g_count, (unsigned long long)cursor);
        atomicMax(p.g_count + 3, (unsigned long long)cursor);
      }
    }
  }
}

}  // namespace glop
