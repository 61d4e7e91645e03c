// kmp.cuh -- K4: chunk-parallel KMP (kmp_search, kmp.hpp:41-69) with the
// reference's exact comparison count.
//
// The reference's failure-function loop is replayed on the host into a DFA
// over (state, byte): entry = next state (13 bits) | match << 13 |
// comparisons << 14, so the sequential comparison count is reproduced step
// by step.  Each of the 512 threads of a CTA owns 144 consecutive END
// positions of a 73,728-byte tile (144 = 9 x 16 bytes: the 32 lanes' LDS.128
// hit distinct banks); the state at its first position is recovered by a
// warm-up over the previous m-1 bytes (the KMP state depends only on them).
// In state 0 a byte other than p[0] costs exactly one comparison and keeps
// state 0, so a thread skips 16-byte groups without p[0] (SWAR test on the
// registers of one LDS.128) and jumps to the next p[0] inside a group; only
// bytes after a p[0] walk the DFA.  Tiles stream HBM -> shared memory by
// 1-D TMA (cp.async.bulk) into a 2-stage ring; matches are ordered per tile
// (shared-memory bitonic sort of the few keys) and laid out by the tile
// directory (tile_prefix_kernel + gather_kernel).
#pragma once
#include <type_traits>

#include "glop_kernels.cuh"

namespace glop {

constexpr int kK2Threads = 512;
constexpr uint32_t kK2Chunk = 144;                   // end positions per thread
constexpr uint32_t kK2Tile = kK2Chunk * kK2Threads;  // 73,728
constexpr uint32_t kK2Pre = 64;                      // warm-up bytes kept before the tile
constexpr uint32_t kK2Stage = kK2Pre + kK2Tile + 16;
constexpr uint32_t kK2HitCap = 1024;                 // match keys per tile in smem
constexpr uint32_t kK2SmemDfaMax = 48;               // patterns up to 48 bytes keep the DFA in smem

struct K2Smem {
  static constexpr uint32_t kBars = 2 * kK2Stage;
  static constexpr uint32_t kMisc = kBars + 16;
  static constexpr uint32_t kKeys = kMisc + 16;
  static constexpr uint32_t kDfa = kKeys + kK2HitCap * 8;
};

struct K2Params {
  const uint8_t* text;
  unsigned long long n, end_lim, base;  // ends (last byte of a match) < end_lim
  uint32_t m, num_tiles, p0;
  const uint32_t* dfa;                  // m x 256
  unsigned long long* staging;
  unsigned long long staging_cap;
  unsigned long long* g_count;
  TileDir* dir;
  unsigned int* g_flags;
  unsigned long long* comparisons;
  int mode;                             // 0: per-tile order; 1: global keys (fallback)
  unsigned long long* keys;
  unsigned long long keys_cap;
};

// TMA window: dst[0, bytes) <- A[lo, lo + bytes) clipped to [a, a + n)
// (lo may be negative); partial 16-byte granules by the issuing thread.
__device__ __forceinline__ void k2_issue(uint8_t* dst, uint64_t* bar, const uint8_t* A, uint32_t a,
                                         unsigned long long n, long long lo, uint32_t bytes) {
  const long long hi = lo + bytes;
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
__global__ void __launch_bounds__(kK2Threads, 1) kmp2_kernel(const K2Params p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t tid = threadIdx.x;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + K2Smem::kBars);
  uint32_t* s_misc = reinterpret_cast<uint32_t*>(smem + K2Smem::kMisc);
  unsigned long long* s_keys = reinterpret_cast<unsigned long long*>(smem + K2Smem::kKeys);
  uint32_t* s_dfa = reinterpret_cast<uint32_t*>(smem + K2Smem::kDfa);
  if (kSmemDfa)
    for (uint32_t i = tid; i < p.m * 64; i += kK2Threads)
      reinterpret_cast<uint4*>(s_dfa)[i] = reinterpret_cast<const uint4*>(p.dfa)[i];
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    s_misc[0] = 0;
    s_misc[1] = 0;
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t* D = kSmemDfa ? s_dfa : p.dfa;
  const uint32_t a = (uint32_t)((uintptr_t)p.text & 15);
  const uint8_t* A = p.text - a;  // 16-aligned; text position x is A[x + a]
  const unsigned long long e_end = p.end_lim + a;  // end positions, A coordinates
  if (tid == 0)
    for (uint32_t s = 0; s < 2; ++s) {
      const uint32_t t = blockIdx.x + s * gridDim.x;
      if (t < p.num_tiles)
        k2_issue(smem + s * kK2Stage, &bars[s], A, a, p.n, (long long)t * kK2Tile - kK2Pre, kK2Stage);
    }
  const uint32_t x4 = p.p0 * 0x01010101u, m = p.m;
  unsigned long long cmp_total = 0;
  for (uint32_t k = 0;; ++k) {
    const uint32_t t = blockIdx.x + k * gridDim.x;
    if (t >= p.num_tiles) break;
    const uint32_t stage = k & 1;
    mbar_wait(&bars[stage], (k >> 1) & 1);
    const uint8_t* win = smem + stage * kK2Stage;
    const unsigned long long tT = (unsigned long long)t * kK2Tile;
    // window byte y holds A[tT - kK2Pre + y]
    auto abyte = [&](unsigned long long x) -> uint32_t {  // A coordinate, a <= x < a + n
      const long long y = (long long)(x - tT) + kK2Pre;
      return (y >= 0 && y < (long long)kK2Stage) ? win[y] : __ldg(A + x);
    };
    auto record = [&](unsigned long long x) {  // match ending at A coordinate x
      if (p.mode == 0) {
        const uint32_t slot = atomicAdd(&s_misc[k & 1], 1u);
        if (slot < kK2HitCap) s_keys[slot] = x - tT;
      } else {
        const unsigned long long slot = atomicAdd(p.g_count, 1ull);
        if (slot < p.keys_cap) p.keys[slot] = p.base + x - a + 1 - m;
      }
    };
    unsigned long long c0 = tT + (unsigned long long)tid * kK2Chunk;
    if (c0 < a) c0 = a;
    const unsigned long long c1 = min(tT + (unsigned long long)(tid + 1) * kK2Chunk, e_end);
    // Walks window bytes [yf, yt) from state j (window byte y is A coordinate
    // tT - kK2Pre + y); in state 0 only p[0] bytes (found 16 at a time) step
    // the DFA.  kCount: add the reference's comparisons and record matches
    // (the warm-up does neither).
    auto walk = [&](auto kCount, uint32_t yf, uint32_t yt, uint32_t& j, unsigned long long& cmp) {
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
          if (decltype(kCount)::value) {
            cmp += e >> 14;
            if (e & 0x2000u) record(tT - kK2Pre + g + kk);
          }
          j = e & 0x1FFFu;
          ++kk;
        }
      }
    };
    if (tid == 0 && p.mode == 0) s_misc[(k + 1) & 1] = 0;  // the next tile's match counter
    if (c0 < c1) {
      const uint32_t y0 = (uint32_t)(c0 - tT) + kK2Pre, y1 = (uint32_t)(c1 - tT) + kK2Pre;
      // warm-up: the state at c0 from the m-1 bytes before it (clamped to the text start)
      uint32_t j = 0;
      unsigned long long cmp = 0;
      const unsigned long long wlo = c0 - min(c0 - a, (unsigned long long)(m - 1));
      if (wlo + kK2Pre >= tT) {
        walk(std::false_type{}, (uint32_t)(wlo + kK2Pre - tT), y0, j, cmp);
      } else {  // long patterns: warm-up bytes before the window
        for (unsigned long long x = wlo; x < c0; ++x) {
          const uint32_t b = abyte(x);
          if (j != 0 || b == p.p0) j = D[j * 256 + b] & 0x1FFFu;
        }
      }
      walk(std::true_type{}, y0, y1, j, cmp);
      cmp_total += cmp;
    }
    __syncthreads();
    if (tid == 0) {
      const uint32_t tn = t + 2 * gridDim.x;
      if (tn < p.num_tiles) {
        fence_proxy_async();
        k2_issue(smem + stage * kK2Stage, &bars[stage], A, a, p.n, (long long)tn * kK2Tile - kK2Pre, kK2Stage);
      }
    }
    if (p.mode != 0) continue;
    const uint32_t nh = s_misc[k & 1];
    if (nh == 0) {  // common case: no match in the tile, no further barrier
      if (tid == 0) p.dir[t] = TileDir{0ull, 0u, 0u};
      continue;
    }
    const bool over = nh > kK2HitCap;
    if (!over && nh > 1) {
      uint32_t P = 1;
      while (P < nh) P <<= 1;
      for (uint32_t y = nh + tid; y < P; y += kK2Threads) s_keys[y] = ~0ull;
      __syncthreads();
      for (uint32_t kk = 2; kk <= P; kk <<= 1)
        for (uint32_t jj = kk >> 1; jj > 0; jj >>= 1) {
          for (uint32_t x = tid; x < P; x += kK2Threads) {
            const uint32_t y = x ^ jj;
            if (y > x) {
              const unsigned long long u = s_keys[x], w = s_keys[y];
              if ((u > w) == ((x & kk) == 0)) s_keys[x] = w, s_keys[y] = u;
            }
          }
          __syncthreads();
        }
    }
    if (tid == 0) {
      const unsigned long long slot = atomicAdd(p.g_count, (unsigned long long)nh);
      p.dir[t] = TileDir{slot, nh, over ? 1u : 0u};
      if (over) atomicOr(p.g_flags, 1u);
      s_misc[2] = (uint32_t)slot;
      s_misc[3] = (uint32_t)(slot >> 32);
    }
    __syncthreads();
    const unsigned long long slot = (unsigned long long)s_misc[2] | ((unsigned long long)s_misc[3] << 32);
    if (!over && slot + nh <= p.staging_cap)
      for (uint32_t h = tid; h < nh; h += kK2Threads) p.staging[slot + h] = p.base + tT + s_keys[h] - a + 1 - m;
    __syncthreads();
  }
  for (int o = 16; o; o >>= 1) cmp_total += __shfl_xor_sync(0xffffffffu, cmp_total, o);
  if ((tid & 31) == 0 && cmp_total) atomicAdd(p.comparisons, cmp_total);
}

}  // namespace glop
