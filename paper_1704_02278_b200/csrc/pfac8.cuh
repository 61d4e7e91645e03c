// pfac8.cuh -- K1 fast path: PFAC for automata whose outputs all lie at depth
// >= 8 (every pattern prefix has 8 bytes; the north_star's "8-character
// truncated prefixes").  Same result as pfac_scan (scan.hpp:113-202) and the
// general kernel in glop_kernels.cuh; leaner per byte:
//
//  * 32 warps per SM, each with a private double-buffered 2 KB TMA ring
//    (cp.async.bulk + mbarrier), tiles assigned round-robin inside the CTA's
//    contiguous range so the tile directory needs no producer id.
//  * Level 1, aligned q-gram sampling: every match start c has, for the
//    unique d in 1..4 with c + d = 0 (mod 4), the pattern's 4-gram at offset d
//    sitting in an aligned text word.  One conflict-free LDS.32 and one hashed
//    d-mask probe per 4 text bytes; no unaligned extraction.
//  * Words with a non-empty d-mask go (in text order) into a 64-entry per-warp
//    ring; full 32-entry rounds are drained: the 8-byte key of each candidate
//    c = 4i - d is assembled from words i-1, i, i+1 with constant funnel
//    shifts and tested in a 2^18-bit prefix bitmap.
//  * Bitmap survivors probe the exact J=8 jump table (generalised RootJump,
//    scan.hpp:81-108) in global memory (L2-resident) and, for patterns longer
//    than 8 bytes, continue the trie walk (scan.hpp:142-168).
//  * Hits of a tile are warp-sorted in shared memory and appended to the
//    warp's staging region; one 8-byte directory record per tile.
#pragma once
#include "glop_kernels.cuh"

namespace glop {

constexpr int kP8Warps = 32;
constexpr int kP8Threads = kP8Warps * 32;
constexpr uint32_t kP8Tile = 2048;                 // owned starts per tile (TMA unit)
constexpr uint32_t kP8Stage = kP8Tile + 16;        // + words 512..515 (halo)
constexpr uint32_t kP8Ring = 128;                  // queue entries per warp (power of 2)
constexpr uint32_t kP8Hits = 64;                   // hit keys per warp in smem
constexpr uint32_t kP8DmaskBytes = 1u << 15;

struct P8Dir {
  uint32_t cursor;  // offset of the tile's hits in its warp's staging region
  uint32_t count;
};

struct P8Layout {
  uint32_t bufs, bars, ring, hits, nh, dmask, bm2, cls, total;
};

__host__ __device__ inline P8Layout make_p8_layout() {
  P8Layout L;
  uint32_t o = 0;
  L.bufs = o; o += kP8Warps * 2 * kP8Stage;
  L.bars = o; o += kP8Warps * 2 * 8;
  L.ring = o; o += kP8Warps * kP8Ring * 4;
  L.hits = o; o += kP8Warps * kP8Hits * 8;
  L.nh = o; o += kP8Warps * 4;
  L.dmask = align16(o); o = L.dmask + kP8DmaskBytes;
  L.bm2 = o; o += kBm2Bytes;
  L.cls = o; o += 256;
  L.total = o;
  return L;
}

struct P8Params {
  const uint8_t* text;
  unsigned long long n, own, base;
  uint32_t num_tiles;
  uint32_t per;                  // tiles per CTA (contiguous range)
  int mode;                      // 0 ordered staging; 1 global keys
  DevHit* staging;
  unsigned long long region;     // staging records per (CTA, warp)
  P8Dir* dir;                    // one record per tile
  unsigned long long* g_count;   // [0] total hits, [1] flags, [2] max region use, [3] mode-1 slots
  unsigned long long* keys;      // mode 1
  unsigned long long keys_cap;
  const uint8_t* dmask8;         // 2^15 d-masks (bit d-1: gram at pattern offset d)
};

// Region (staging area / producing warp) of tile t under the round-robin
// assignment below.
__host__ __device__ __forceinline__ uint32_t p8_region(uint32_t t, uint32_t per) {
  const uint32_t b = t / per;
  return b * kP8Warps + (t - b * per) % kP8Warps;
}

// 1-D TMA bulk copy of aligned text A[lo, lo + kP8Stage) (clipped to the
// valid range [a, a + n)) into dst; bytes outside 16-byte granules are copied
// by the issuing lane.  One arrival (with tx bytes) on bar.
__device__ __forceinline__ void p8_issue(uint8_t* dst, uint64_t* bar, const uint8_t* A, uint32_t a,
                                         unsigned long long n, unsigned long long lo) {
  const unsigned long long hi = lo + kP8Stage;
  const unsigned long long vlo = lo > a ? lo : a, vhi = hi < a + n ? hi : a + n;
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

// Sorts the warp's nb buffered hit keys (tile position << 32 | pattern id)
// and writes them as hits to dst (nullptr: the warp's staging region is full;
// the host grows it and reruns).  nb > kP8Hits means keys were dropped: the
// scan is flagged for the exact global-key fallback.  Whole warp.
__device__ __noinline__ uint32_t p8_flush(unsigned long long* hk, uint32_t nb, uint32_t lane, DevHit* dst,
                                          unsigned long long off0, const uint32_t* pid_len,
                                          unsigned long long* g_count) {
  if (nb > kP8Hits) {
    if (lane == 0) {
      atomicAdd(g_count, (unsigned long long)nb);
      atomicOr(reinterpret_cast<unsigned int*>(g_count + 1), 1u);
    }
    return 0;
  }
  warp_sort_keys(hk, nb, lane);
  if (dst)
    for (uint32_t h = lane; h < nb; h += 32) {
      const unsigned long long key = hk[h];
      DevHit out;
      out.offset = off0 + (key >> 32);
      out.pid = (uint32_t)key;
      out.len = __ldg(pid_len + out.pid);
      dst[h] = out;
    }
  __syncwarp();
  return nb;
}

template <bool kWalk, typename Entry>
__global__ void __launch_bounds__(kP8Threads, 1)
    pfac8_kernel(const DevTrie tr, const P8Params p, const P8Layout L) {
  using ET = EntryTraits<Entry>;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint8_t* s_dmask = smem + L.dmask;
  const uint32_t* s_bm2 = reinterpret_cast<const uint32_t*>(smem + L.bm2);
  const uint8_t* s_cls = smem + L.cls;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars) + warp * 2;
  uint8_t* bufs = smem + L.bufs + (size_t)warp * 2 * kP8Stage;
  uint32_t* q = reinterpret_cast<uint32_t*>(smem + L.ring) + warp * kP8Ring;
  unsigned long long* hk = reinterpret_cast<unsigned long long*>(smem + L.hits) + warp * kP8Hits;
  uint32_t* s_nh = reinterpret_cast<uint32_t*>(smem + L.nh) + warp;

  const uint32_t t_begin = min(blockIdx.x * p.per, p.num_tiles);
  const uint32_t t_end = min(t_begin + p.per, p.num_tiles);
  {
    const uint4* s = reinterpret_cast<const uint4*>(p.dmask8);
    uint4* d = reinterpret_cast<uint4*>(smem + L.dmask);
    for (uint32_t i = tid; i < kP8DmaskBytes / 16; i += kP8Threads) d[i] = s[i];
    s = reinterpret_cast<const uint4*>(tr.bm2);
    d = reinterpret_cast<uint4*>(smem + L.bm2);
    for (uint32_t i = tid; i < kBm2Bytes / 16; i += kP8Threads) d[i] = s[i];
    if (kWalk && tid < 16) reinterpret_cast<uint4*>(smem + L.cls)[tid] = reinterpret_cast<const uint4*>(tr.cls)[tid];
    if (lane < 2) mbar_init(&bars[lane], 1);
    if (lane == 0) *s_nh = 0;
    if (tid == 0) fence_mbar_init();
  }
  __syncthreads();
  const uint32_t a = (uint32_t)((uintptr_t)p.text & 15);
  const uint8_t* A = p.text - a;
  if (lane == 0)
    for (uint32_t b = 0; b < 2; ++b) {
      const uint32_t t = t_begin + warp + b * kP8Warps;
      if (t < t_end) p8_issue(bufs + b * kP8Stage, &bars[b], A, a, p.n, (unsigned long long)t * kP8Tile);
    }
  const unsigned long long own_end = p.own + a, n_end = p.n + a;  // aligned coordinates
  const uint32_t gw = blockIdx.x * kP8Warps + warp;
  const unsigned long long region_base = (unsigned long long)gw * p.region;
  const uint32_t cap_log2 = tr.jump_cap_log2, hmask = (1u << cap_log2) - 1;
  const uint32_t lmax = tr.lmax, C = tr.C;
  const Entry* T = reinterpret_cast<const Entry*>(tr.table);
  uint32_t cursor = 0;
  uint32_t ltmask;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(ltmask));

  for (uint32_t k = 0;; ++k) {
    const uint32_t t = t_begin + warp + k * kP8Warps;
    if (t >= t_end) break;
    const uint32_t b = k & 1;
    mbar_wait(&bars[b], (k >> 1) & 1);
    const uint8_t* sb = bufs + b * kP8Stage;
    const uint32_t* sw = reinterpret_cast<const uint32_t*>(sb);
    const unsigned long long tA = (unsigned long long)t * kP8Tile;
    const uint32_t s_hi = (uint32_t)min(own_end - tA, (unsigned long long)kP8Tile);
    const uint32_t avail = (uint32_t)min(n_end - tA, 0x7FFFFFFFull);
    const uint32_t lo = t == 0 ? a : 0;
    const unsigned long long off0 = p.base + tA - a;  // text offset of window byte 0
    const bool edge = lo != 0 || s_hi < kP8Tile || avail < kP8Tile + 8;
    uint32_t seg_n = 0;                              // hits of this tile written so far
    auto flush = [&](uint32_t nb) {
      const bool fits = cursor + seg_n + nb <= p.region;
      seg_n += p8_flush(hk, nb, lane, fits ? p.staging + region_base + cursor + seg_n : nullptr, off0,
                        tr.pid_len, p.g_count);
      if (lane == 0) *s_nh = 0;
      __syncwarp();
    };

    auto emit = [&](uint32_t c, uint32_t pid) {
      if (p.mode == 0) {
        const uint32_t slot = atomicAdd(s_nh, 1u);
        if (slot < kP8Hits) hk[slot] = ((unsigned long long)c << 32) | pid;
      } else {
        const unsigned long long slot = atomicAdd(p.g_count + 3, 1ull);
        if (slot < p.keys_cap) p.keys[slot] = ((off0 + c) << 24) | pid;
      }
    };
    auto emit_state = [&](uint32_t c, uint32_t st) {
      for (uint32_t o = __ldg(tr.out_off + st), oe = __ldg(tr.out_off + st + 1); o < oe; ++o)
        emit(c, __ldg(tr.out_pid + o));
    };
    // exact check of candidate start c with 8-byte key (lo32, hi32)
    auto exact = [&](uint32_t c, uint32_t klo, uint32_t khi) {
      const unsigned long long key = (unsigned long long)klo | ((unsigned long long)khi << 32);
      for (uint32_t h = jump_slot(key, cap_log2);; h = (h + 1) & hmask) {
        const JumpEntry e = tr.jump[h];
        if (!e.state1) return;
        if (e.key != key) continue;
        uint32_t st = e.state1 - 1;
        if (e.out != kOutNone) {
          if (e.out == kOutMany) emit_state(c, st);
          else emit(c, e.out);
        }
        if (kWalk && lmax > 8) {  // deeper levels: scan.hpp:142-168
          for (uint32_t j = c + 8; j < avail; ++j) {
            const uint32_t byte = j < kP8Stage ? sb[j] : __ldg(p.text + (tA + j - a));
            const uint32_t x = __ldg(T + st * C + s_cls[byte]);
            if (!x) break;
            st = x & ET::kMask;
            if (x & ET::kFlag) emit_state(c, st);
          }
        }
        return;
      }
    };

    // 4 chunks of 512 bytes: lane l samples tile words 128 it + 4 l + 1 .. + 4
    // (candidates 0..2047 of the tile), then the chunk's candidate words are
    // compacted (text order) into q and checked 32 at a time.
#pragma unroll 1
    for (uint32_t it = 0; it < 4; ++it) {
      const uint4 v = reinterpret_cast<const uint4*>(sb)[32 * it + lane];
      const uint32_t wn = sw[128 * it + 128];
      uint32_t w4 = __shfl_down_sync(0xffffffffu, v.x, 1);
      if (lane == 31) w4 = wn;
      const uint32_t m0 = s_dmask[qgram_bucket(v.y, 4)], m1 = s_dmask[qgram_bucket(v.z, 4)];
      const uint32_t m2 = s_dmask[qgram_bucket(v.w, 4)], m3 = s_dmask[qgram_bucket(w4, 4)];
      if (!__ballot_sync(0xffffffffu, (m0 | m1 | m2 | m3) != 0)) continue;
      // number of candidate words of this lane (d-masks are < 16, so adding
      // 0x7F to each byte sets its top bit iff the byte is non-zero)
      const uint32_t packed = __byte_perm(m0 | (m1 << 8), m2 | (m3 << 8), 0x5410);
      const uint32_t cnt = __popc((packed + 0x7F7F7F7Fu) & 0x80808080u);
      const uint32_t b0 = __ballot_sync(0xffffffffu, cnt & 1), b1 = __ballot_sync(0xffffffffu, cnt & 2),
                     b2 = __ballot_sync(0xffffffffu, cnt & 4);
      const uint32_t tot = __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
      {
        uint32_t* qp = q + __popc(b0 & ltmask) + 2 * __popc(b1 & ltmask) + 4 * __popc(b2 & ltmask);
        const uint32_t wbase = (128 * it + 4 * lane + 1) << 4;
        if (m0) *qp++ = wbase + m0;
        if (m1) *qp++ = wbase + 16 + m1;
        if (m2) *qp++ = wbase + 32 + m2;
        if (m3) *qp = wbase + 48 + m3;
      }
      __syncwarp();
#pragma unroll 1
      for (uint32_t r = 0; r < tot; r += 32) {
        // ---- 8-byte keys of the candidates -> prefix bitmap
        const uint32_t e = r + lane < tot ? q[r + lane] : 16u;  // idle lanes: word 1, no candidates
        const uint32_t i = e >> 4;
        uint32_t m = e & 15u;
        const uint32_t w0 = sw[i - 1], w1 = sw[i], w2 = sw[i + 1];
        if (edge) {
#pragma unroll
          for (uint32_t d = 1; d <= 4; ++d) {
            const uint32_t c = 4 * i - d;
            if (c < lo || c >= s_hi || c + 8 > avail) m &= ~(1u << (d - 1));
          }
        }
        uint32_t surv = 0;
#pragma unroll
        for (uint32_t d = 1; d <= 4; ++d) {
          const uint32_t x = prefix_hash32(__funnelshift_r(w0, w1, 32 - 8 * d), __funnelshift_r(w1, w2, 32 - 8 * d));
          const uint32_t word = s_bm2[x >> (32 - kBm2Log2 + 5)];
          surv |= (__funnelshift_r(word, 0u, x >> (32 - kBm2Log2)) & (m >> (d - 1)) & 1u) << (d - 1);
        }
        const uint32_t runmask = __ballot_sync(0xffffffffu, surv != 0);
        if (!runmask) continue;
        // ---- exact check of the survivors; a pass that overflows the hit
        // buffer is dropped and replayed lane by lane (lanes hold ascending
        // candidates), flushing in between
        const uint32_t nb0 = *s_nh;  // <= kP8Hits / 2
        uint32_t mask = runmask, redo = 0;
        bool first = true;
        for (;;) {
          if ((mask >> lane) & 1u) {
            uint32_t sv = surv;
            while (sv) {
              const uint32_t d = __ffs(sv);  // 1..4
              sv &= sv - 1;
              const uint32_t sh = 32 - 8 * d;
              exact(4 * i - d, __funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh));
            }
          }
          __syncwarp();
          const uint32_t nb = *s_nh;
          __syncwarp();
          if (p.mode == 0) {
            if (first && nb > kP8Hits) {
              if (lane == 0) *s_nh = nb0;
              __syncwarp();
              redo = runmask;
            } else if (nb > kP8Hits / 2) {
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
    if (p.mode == 0) {
      __syncwarp();
      const uint32_t nb = *s_nh;
      if (nb) {
        __syncwarp();
        flush(nb);
      }
    }
    // buffer b is free: refill it with this warp's tile k + 2
    __syncwarp();
    if (lane == 0) {
      if (p.mode == 0) {
        p.dir[t] = P8Dir{cursor, seg_n};
        if (seg_n) atomicAdd(p.g_count, (unsigned long long)seg_n);
      }
      const uint32_t tn = t + 2 * kP8Warps;
      if (tn < t_end) {
        fence_proxy_async();
        p8_issue(bufs + b * kP8Stage, &bars[b], A, a, p.n, (unsigned long long)tn * kP8Tile);
      }
    }
    cursor += seg_n;
  }
  if (p.mode == 0 && lane == 0 && cursor) atomicMax(p.g_count + 2, (unsigned long long)cursor);
}

// ---- P8 tile directory -> ordered output (same scheme as seg_* above)
__global__ void __launch_bounds__(1024) p8_reduce_kernel(const P8Dir* dir, unsigned long long nseg,
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

__global__ void __launch_bounds__(1024) p8_gather_kernel(const P8Dir* dir, unsigned long long nseg,
                                                         const unsigned long long* block_prefix, uint32_t per,
                                                         unsigned long long region, const DevHit* staging,
                                                         DevHit* out) {
  __shared__ uint32_t ws[32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const unsigned long long b = (unsigned long long)blockIdx.x * kSegPerBlock + tid * kSegPerThread;
  uint32_t c[kSegPerThread], s = 0;
  for (uint32_t i = 0; i < kSegPerThread; ++i) {
    c[i] = b + i < nseg ? dir[b + i].count : 0;
    s += c[i];
  }
  uint32_t incl = s;
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
    const unsigned long long t = b + i;
    const unsigned long long src = (unsigned long long)p8_region((uint32_t)t, per) * region + dir[t].cursor;
    for (uint32_t h = 0; h < c[i]; ++h) out[dst + h] = staging[src + h];
    dst += c[i];
  }
}

}  // namespace glop
