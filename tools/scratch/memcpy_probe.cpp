#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <string>
#include <cstdlib>
struct A { size_t off, line; unsigned id; std::string name; unsigned len; bool v; };
int main() {
  size_t n = 1ull << 30;
  char* src = (char*)malloc(n); char* dst = (char*)malloc(n);
  memset(src, 1, n); memset(dst, 2, n);
  for (int T : {1, 4, 8, 16}) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> p; size_t per = n / T;
    for (int t = 0; t < T; ++t) p.emplace_back([=]{ memcpy(dst + t*per, src + t*per, per); });
    for (auto& x : p) x.join();
    double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("T=%d %.1f GB/s\n", T, n / s / 1e9);
  }
  auto t0 = std::chrono::steady_clock::now();
  std::vector<A> v; v.reserve(2000000);
  for (int i = 0; i < 2000000; ++i) { A a; a.off = i; a.line = 0; a.id = i % 1000; a.name = "r" + std::to_string(i % 1000); a.len = 8; a.v = true; v.push_back(std::move(a)); }
  double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  printf("2M alerts: %.1f ms\n", s * 1e3);
}
