#include <chrono>
#include <cstdio>
#include <string>
#include <vector>
#include <thread>
#include <cstring>
#include <memory>
struct Alert { size_t offset = 0, line = 0; unsigned rule_id = 0; std::string rule_name; unsigned pattern_len = 0; bool verified = false; };
int main() {
  const size_t n = 2022985;
  std::vector<std::string> names(1000); for (int i = 0; i < 1000; ++i) names[i] = "r" + std::to_string(i);
  for (int rep = 0; rep < 3; ++rep) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<Alert> v(n);
    auto t1 = std::chrono::steady_clock::now();
    unsigned T = std::thread::hardware_concurrency();
    std::vector<std::thread> p;
    for (unsigned t = 0; t < T; ++t) p.emplace_back([&, t] { for (size_t i = t * n / T; i < (t + 1) * n / T; ++i) { v[i].offset = i; v[i].rule_id = i % 1000; v[i].rule_name = names[i % 1000]; v[i].pattern_len = 8; v[i].verified = true; } });
    for (auto& x : p) x.join();
    auto t2 = std::chrono::steady_clock::now();
    { std::vector<Alert> w; w.swap(v); }
    auto t3 = std::chrono::steady_clock::now();
    printf("construct %.1f fill %.1f destroy %.1f ms\n", std::chrono::duration<double,std::milli>(t1-t0).count(), std::chrono::duration<double,std::milli>(t2-t1).count(), std::chrono::duration<double,std::milli>(t3-t2).count());
  }
}
