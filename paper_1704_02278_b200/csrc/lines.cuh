// lines.cuh -- device LineIndex (reference LineIndex,
// verify.hpp:40-64): the 1-based line of an offset is 1 + the number of LF
// bytes before it (an LF belongs to the line it ends).  One HBM pass counts
// LFs per 4 KB block (SWAR byte compare on 16-byte loads), a device scan turns
// the counts into block prefixes, and one warp per queried offset adds the
// LFs between its block start and the offset.
#pragma once
#include "glop_kernels.cuh"

namespace glop {

constexpr uint32_t kLineBlock = 4096;

__device__ __forceinline__ uint32_t lf_count_word(uint32_t w) {
  const uint32_t t = w ^ 0x0A0A0A0Au;                     // LF bytes -> 0
  return __popc(~(((t & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | t | 0x7F7F7F7Fu));  // exact zero-byte count
}

// LFs in text[lo, hi) (text 16-aligned at `A`, positions relative to A).
__device__ __forceinline__ uint32_t lf_count_range(const uint8_t* A, unsigned long long lo, unsigned long long hi,
                                                   uint32_t lane, uint32_t lanes) {
  uint32_t c = 0;
  const unsigned long long a16 = (lo + 15) & ~15ull, b16 = hi & ~15ull;
  if (a16 >= b16) {
    for (unsigned long long x = lo + lane; x < hi; x += lanes) c += A[x] == '\n';
    return c;
  }
  for (unsigned long long x = lo + lane; x < a16; x += lanes) c += A[x] == '\n';
  for (unsigned long long x = b16 + lane; x < hi; x += lanes) c += A[x] == '\n';
  for (unsigned long long x = a16 + 16ull * lane; x < b16; x += 16ull * lanes) {
    const uint4 v = *reinterpret_cast<const uint4*>(A + x);
    c += lf_count_word(v.x) + lf_count_word(v.y) + lf_count_word(v.z) + lf_count_word(v.w);
  }
  return c;
}

// counts[b] = LFs in block b of text[0, n) (A = text - a, blocks in A coordinates).
__global__ void __launch_bounds__(256) lf_block_count_kernel(const uint8_t* A, uint32_t a, unsigned long long n,
                                                             unsigned long long nblocks, unsigned long long* counts) {
  const uint32_t lane = threadIdx.x & 31;
  for (unsigned long long b = (blockIdx.x * 256ull + threadIdx.x) / 32; b < nblocks;
       b += (unsigned long long)gridDim.x * 8) {
    const unsigned long long lo = max(b * kLineBlock, (unsigned long long)a);
    const unsigned long long hi = min((b + 1) * kLineBlock, a + n);
    uint32_t c = lo < hi ? lf_count_range(A, lo, hi, lane, 32) : 0u;
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) counts[b] = c;
  }
}

// lines[i] = 1 + LFs in text[0, offsets[i] - base) (+ *line_base: LFs of
// earlier streamed chunks) (warp per offset).
__global__ void __launch_bounds__(256) lines_of_kernel(const uint8_t* A, uint32_t a, unsigned long long base,
                                                       const unsigned long long* prefix, const void* recs,
                                                       uint32_t stride, unsigned long long count,
                                                       unsigned long long* lines,
                                                       const unsigned long long* line_base) {
  const uint32_t lane = threadIdx.x & 31;
  const unsigned long long lb = line_base ? *line_base : 0;
  for (unsigned long long i = (blockIdx.x * 256ull + threadIdx.x) / 32; i < count;
       i += (unsigned long long)gridDim.x * 8) {
    const unsigned long long off =
        *reinterpret_cast<const unsigned long long*>(static_cast<const uint8_t*>(recs) + i * stride) - base + a;
    const unsigned long long b = off / kLineBlock;
    uint32_t c = lf_count_range(A, max(b * kLineBlock, (unsigned long long)a), off, lane, 32);
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) lines[i] = prefix[b] + c + 1 + lb;
  }
}

// *acc += LFs of the whole text (last block prefix + last block count).
__global__ void lf_total_add_kernel(const unsigned long long* counts, const unsigned long long* prefix,
                                    unsigned long long nblocks, unsigned long long* acc) {
  *acc += prefix[nblocks - 1] + counts[nblocks - 1];
}

// Lines of offsets into an empty text: 1 (+ *line_base).
__global__ void lines_fill_kernel(unsigned long long* lines, unsigned long long count,
                                  const unsigned long long* line_base) {
  const unsigned long long lb = line_base ? *line_base : 0;
  for (unsigned long long i = threadIdx.x; i < count; i += blockDim.x) lines[i] = 1 + lb;
}

}  // namespace glop
