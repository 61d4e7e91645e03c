// scratch: copy-kernel variants for the pageable staging copy
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
int main() {
  size_t n = 4ull << 30;
  uint8_t* a = (uint8_t*)aligned_alloc(4096, n); uint8_t* b = (uint8_t*)aligned_alloc(4096, n);
  memset(a, 1, n); memset(b, 2, n);
  for (unsigned T : {8u, 12u, 16u}) {
    double c512 = run(T, n, [&](size_t lo, size_t hi) {
      for (size_t i = lo; i < hi; i += 256) { for (int k = 0; k < 4; ++k) _mm512_stream_si512((__m512i*)(b + i + 64 * k), _mm512_loadu_si512((a + i + 64 * k))); } _mm_sfence(); });
    double c512p = run(T, n, [&](size_t lo, size_t hi) {
      for (size_t i = lo; i < hi; i += 256) { _mm_prefetch((const char*)a + i + 2048, _MM_HINT_T0); _mm_prefetch((const char*)a + i + 2048 + 64, _MM_HINT_T0); _mm_prefetch((const char*)a + i + 2048 + 128, _MM_HINT_T0); _mm_prefetch((const char*)a + i + 2048 + 192, _MM_HINT_T0);
        for (int k = 0; k < 4; ++k) _mm512_stream_si512((__m512i*)(b + i + 64 * k), _mm512_loadu_si512((a + i + 64 * k))); } _mm_sfence(); });
    double c256p = run(T, n, [&](size_t lo, size_t hi) {
      for (size_t i = lo; i < hi; i += 128) { _mm_prefetch((const char*)a + i + 2048, _MM_HINT_T0); _mm_prefetch((const char*)a + i + 2048 + 64, _MM_HINT_T0);
        for (int k = 0; k < 4; ++k) _mm256_stream_si256((__m256i*)(b + i + 32 * k), _mm256_loadu_si256((__m256i*)(a + i + 32 * k))); } _mm_sfence(); });
    double movsb = run(T, n, [&](size_t lo, size_t hi) { void* d = b + lo; const void* s = a + lo; size_t c = hi - lo; asm volatile("rep movsb" : "+D"(d), "+S"(s), "+c"(c) : : "memory"); });
    double m = run(T, n, [&](size_t lo, size_t hi) { memcpy(b + lo, a + lo, hi - lo); });
    printf("T=%2u nt512 %.1f nt512+pf %.1f nt256+pf %.1f movsb %.1f memcpy %.1f GB/s\n", T, c512, c512p, c256p, movsb, m);
  }
}
