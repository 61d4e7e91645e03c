// pipeline.cuh -- the device half of run_engine_scan's PFAC branch
// (pipeline.hpp:86-97) after pfac8_kernel, enqueued without host round trips:
//
//   pfac8_kernel        per-warp staging regions (already in text order)
//                       (its grid also zeroes the per-pattern counts)
//   p8_keep_kernel      stage 2 only (some pattern longer than the prefix):
//                       the suffix compare of verify_hits (verify.hpp:78-87)
//                       per hit -> keep flags + kept count per region
//   p8_emit_kernel      each CTA a contiguous range of regions, its output
//                       offsets summed from the counts before it (no prefix
//                       launch); stable compaction of the kept hits into alerts in
//                       (offset, rule_id) order (verify.hpp:100-103: the
//                       regions are already sorted), the optional ordered hit
//                       list, and the per-pattern alert histogram
//
// The host reads one 64-byte status block at the end (totals, the scan's
// overflow flags, verify's logic_error flag); a scan that overflowed a
// staging region or a hit buffer is redone by the general path.
#pragma once
#include "glop_kernels.cuh"
#include "pfac8.cuh"

namespace glop {

// Status words in the scan's g_count block (u64 each).
enum : uint32_t { kStTotal = 0, kStFlags = 1, kStMaxRegion = 2, kStKeys = 3, kStHits = 4, kStKept = 5,
                  kStVerify = 6 };

// 8 bytes at any alignment from two aligned loads (the caller keeps p + 15
// inside the allocation).
__device__ __forceinline__ unsigned long long load8_any(const uint8_t* p) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const unsigned long long* q = reinterpret_cast<const unsigned long long*>(a & ~uintptr_t(7));
  const uint32_t sh = (uint32_t)(a & 7) * 8;
  const unsigned long long lo = __ldg(q);
  return sh ? (lo >> sh) | (__ldg(q + 1) << (64 - sh)) : lo;
}

// text[0, len) == pat[0, len): 8 bytes per step while both reads stay
// inside their buffers (text: [.., t_end); pattern bytes are padded to 16).
__device__ __forceinline__ bool suffix_equal(const uint8_t* t, const uint8_t* t_end, const uint8_t* pat,
                                             unsigned long long len) {
  while (len >= 8 && t + 16 <= t_end) {
    if (load8_any(t) != load8_any(pat)) return false;
    t += 8, pat += 8, len -= 8;
  }
  for (unsigned long long k = 0; k < len; ++k)
    if (t[k] != pat[k]) return false;
  return true;
}

// Stage 2 of verify_hits for hits staged per region: keep[g * region + i]
// and the kept count of region g.  Flag 1 of *vflags: a hit past the end of
// the text or naming an unknown pattern (the reference's logic_error /
// rules.patterns.at(), verify.hpp:76-79).  One CTA per region, grid-stride.
__global__ void __launch_bounds__(256) p8_keep_kernel(const DevRules r, const uint8_t* text,
                                                      unsigned long long base, unsigned long long n,
                                                      const unsigned long long* counts, uint32_t regions,
                                                      unsigned long long region, const DevHit* staging,
                                                      uint8_t* keep, unsigned long long* kcounts,
                                                      unsigned long long* vflags) {
  __shared__ uint32_t s_cnt;
  for (uint32_t g = blockIdx.x; g < regions; g += gridDim.x) {
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    const unsigned long long c = min(counts[g], region);
    const DevHit* src = staging + (unsigned long long)g * region;
    uint8_t* kp = keep + (unsigned long long)g * region;
    uint32_t mine = 0, bad = 0;
    for (unsigned long long i = threadIdx.x; i < c; i += blockDim.x) {
      const DevHit x = src[i];
      uint32_t ok = 0;
      if (x.offset < base || x.offset + x.len > base + n || x.pid >= r.n_patterns) {
        bad = 1;
      } else {
        const unsigned long long pb = r.off[x.pid], plen = r.off[x.pid + 1] - pb;
        if (plen <= r.prefix_len) {
          ok = 1;
        } else if (x.offset + plen <= base + n) {
          const uint8_t* t = text + (x.offset - base);
          ok = suffix_equal(t + x.len, text + n, r.bytes + pb + x.len, plen - x.len);
        }
      }
      kp[i] = (uint8_t)ok;
      mine += ok;
    }
    if (bad) atomicOr(reinterpret_cast<unsigned int*>(vflags), 1u);
    for (uint32_t o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&s_cnt, mine);
    __syncthreads();
    if (threadIdx.x == 0) kcounts[g] = s_cnt;
    __syncthreads();
  }
}

// Region hits -> alerts (+ optionally the ordered hit list).  kStage2:
// compaction by the keep flags at kprefix[g]; otherwise every hit is an
// alert at hprefix[g] + i (all patterns fit in the prefix: verify.hpp:80).
// The per-pattern histogram lives in shared memory (hist_bins = n_patterns,
// flushed once per CTA) when it fits, else global atomics.  Without stage 2
// the bounds / id checks happen here (flag 1 of *vflags).
// Each CTA takes a contiguous range of regions and computes the output
// offsets of its range itself (sums of the hit / kept counts before it), so
// no prefix kernel runs between the scan and this one; CTA 0 also writes the
// totals to the status block (g_status[kStHits], [kStKept]).  The range's
// hits are walked as ONE index space in 1,024-hit chunks (a shared-memory
// prefix of the region counts maps an index to its region), so a CTA spends
// ceil(range hits / 1,024) chunks instead of one chunk per region (the
// per-region loop took 11 us for a 256 MB scan with few hits).
template <bool kStage2>
__global__ void __launch_bounds__(1024) p8_emit_kernel(const DevRules r, unsigned long long base,
                                                       unsigned long long n, const unsigned long long* counts,
                                                       uint32_t regions, unsigned long long region,
                                                       const DevHit* staging, const uint8_t* keep,
                                                       const unsigned long long* kcounts, DevHit* hits_out,
                                                       unsigned long long hit_cap, DevAlert* out,
                                                       unsigned long long alert_cap, unsigned long long* gcounts,
                                                       uint32_t hist_bins, unsigned long long* g_status) {
  extern __shared__ uint32_t hist[];
  __shared__ uint32_t warp_base[32];
  __shared__ uint32_t chunk_total;
  __shared__ unsigned long long s_red[32], s_pre[kRangeMax + 1];
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (uint32_t i = tid; i < hist_bins; i += blockDim.x) hist[i] = 0;
  const uint32_t per = (regions + gridDim.x - 1) / gridDim.x;
  const uint32_t g0 = min(blockIdx.x * per, regions), g1 = min(g0 + per, regions);
  unsigned long long hp = block_sum_counts(counts, g0, region, s_red);
  unsigned long long kp = kStage2 ? block_sum_counts(kcounts, g0, region, s_red) : 0ull;
  if (blockIdx.x == 0) {
    const unsigned long long th = block_sum_counts(counts, regions, region, s_red);
    const unsigned long long tk = kStage2 ? block_sum_counts(kcounts, regions, region, s_red) : 0ull;
    if (tid == 0) {
      g_status[kStHits] = th;
      if (kStage2) g_status[kStKept] = tk;
    }
  }
  unsigned long long* vflags = g_status + kStVerify;
  uint32_t bad = 0;
  for (uint32_t c0 = g0; c0 < g1; c0 += kRangeMax) {  // (one pass with the launch geometries used)
    const uint32_t nr = min(g1 - c0, kRangeMax);
    __syncthreads();  // (the previous pass's prefix is no longer read)
    range_prefix(counts, c0, nr, region, s_pre);
    __syncthreads();
    const unsigned long long total = s_pre[nr];
    for (unsigned long long f0 = 0; f0 < total; f0 += blockDim.x) {
      const unsigned long long f = f0 + tid;
      DevHit x{};
      uint32_t ok = 0;
      if (f < total) {
        uint32_t lo = 0, hi = nr;  // the region j with s_pre[j] <= f < s_pre[j + 1]
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (s_pre[mid] <= f) lo = mid;
          else hi = mid;
        }
        const unsigned long long at = (unsigned long long)(c0 + lo) * region + (f - s_pre[lo]);
        x = staging[at];
        if (hits_out && hp + f < hit_cap) hits_out[hp + f] = x;
        if (kStage2) {
          ok = keep[at];
        } else {
          ok = 1;
          if (x.offset < base || x.offset + x.len > base + n || x.pid >= r.n_patterns) bad = 1, ok = 0;
        }
      }
      unsigned long long dst = hp + f;
      if (kStage2) {  // stable compaction of this chunk: warp counts, one warp scans them
        const uint32_t bal = __ballot_sync(0xffffffffu, ok);
        if (lane == 0) warp_base[w] = __popc(bal);
        __syncthreads();
        if (w == 0) {
          const uint32_t v = lane < blockDim.x / 32 ? warp_base[lane] : 0u;
          uint32_t incl = v;
          for (uint32_t o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          warp_base[lane] = incl - v;
          if (lane == 31) chunk_total = incl;
        }
        __syncthreads();
        dst = kp + warp_base[w] + __popc(bal & ((1u << lane) - 1));
        kp += chunk_total;
        __syncthreads();
      }
      if (ok) {
        if (dst < alert_cap) {
          DevAlert a;
          a.offset = x.offset;
          a.rule_id = x.pid;
          a.pattern_len = (uint32_t)(r.off[x.pid + 1] - r.off[x.pid]);
          out[dst] = a;
        }
        if (hist_bins) atomicAdd(&hist[x.pid], 1u);
        else atomicAdd(gcounts + x.pid, 1ull);
      }
    }
    hp += total;
  }
  if (bad) atomicOr(reinterpret_cast<unsigned int*>(vflags), 1u);
  __syncthreads();
  for (uint32_t i = tid; i < hist_bins; i += blockDim.x)
    if (hist[i]) atomicAdd(gcounts + i, (unsigned long long)hist[i]);
}

// acc[i] += add[i] (per-pattern counts of one streamed chunk).
__global__ void add_u64_kernel(unsigned long long* acc, const unsigned long long* add, uint32_t k) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) acc[i] += add[i];
}

}  // namespace glop
