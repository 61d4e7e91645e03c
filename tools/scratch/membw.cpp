// scratch: host memory bandwidth (read / NT write / NT copy) with T threads
#include <immintrin.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <cstdint>
template <class F> double run(unsigned T, size_t n, F f) {
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> v; size_t per = (n / T) & ~size_t(4095);
  for (unsigned t = 0; t < T; ++t) v.emplace_back([=] { f(t * per, t + 1 == T ? n : (t + 1) * per); });
  for (auto& x : v) x.join();
  return n / std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / 1e9;
}
__attribute__((target("avx2"))) int main(int argc, char** argv) {
  size_t n = 4ull << 30;
  uint8_t* a = (uint8_t*)aligned_alloc(4096, n); uint8_t* b = (uint8_t*)aligned_alloc(4096, n);
  memset(a, 1, n); memset(b, 2, n);
  for (unsigned T : {4u, 8u, 16u}) {
    volatile long sink = 0;
    double r = run(T, n, [&](size_t lo, size_t hi) { __m256i s = _mm256_setzero_si256();
      for (size_t i = lo; i < hi; i += 128) { s = _mm256_add_epi64(s, _mm256_load_si256((__m256i*)(a + i))); s = _mm256_add_epi64(s, _mm256_load_si256((__m256i*)(a + i + 32)));
        s = _mm256_add_epi64(s, _mm256_load_si256((__m256i*)(a + i + 64))); s = _mm256_add_epi64(s, _mm256_load_si256((__m256i*)(a + i + 96))); }
      sink += _mm256_extract_epi64(s, 0); });
    double w = run(T, n, [&](size_t lo, size_t hi) { __m256i z = _mm256_set1_epi8(3);
      for (size_t i = lo; i < hi; i += 128) { _mm256_stream_si256((__m256i*)(b + i), z); _mm256_stream_si256((__m256i*)(b + i + 32), z);
        _mm256_stream_si256((__m256i*)(b + i + 64), z); _mm256_stream_si256((__m256i*)(b + i + 96), z); } _mm_sfence(); });
    double c = run(T, n, [&](size_t lo, size_t hi) {
      for (size_t i = lo; i < hi; i += 128) { for (int k = 0; k < 4; ++k) _mm256_stream_si256((__m256i*)(b + i + 32 * k), _mm256_load_si256((__m256i*)(a + i + 32 * k))); } _mm_sfence(); });
    double m = run(T, n, [&](size_t lo, size_t hi) { memcpy(b + lo, a + lo, hi - lo); });
    printf("T=%2u read %.1f GB/s, NT write %.1f GB/s, NT copy %.1f GB/s, memcpy %.1f GB/s\n", T, r, w, c, m);
  }
}
