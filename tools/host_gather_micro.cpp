// Host random-row gather bandwidth (n=1e6 rows of 100 doubles) by thread count:
//   g++ -O3 -pthread -o /tmp/hg tools/host_gather_micro.cpp && /tmp/hg
#include <cstdio>
#include <cstring>
#include <vector>
#include <thread>
#include <chrono>
#include <random>
#include <algorithm>
#include <cstdint>
int main() {
  const int64_t n = 1000000, p = 100;
  std::vector<double> x(n * p), y(n * p);
  for (int64_t i = 0; i < n * p; ++i) x[i] = i;
  std::vector<int64_t> o(n);
  for (int64_t i = 0; i < n; ++i) o[i] = i;
  std::shuffle(o.begin(), o.end(), std::mt19937_64(1));
  for (int T : {1, 2, 4, 8, 16}) {
    for (int rep = 0; rep < 2; ++rep) {
      auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> th;
      for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
          const int64_t a = n * t / T, b = n * (t + 1) / T;
          for (int64_t i = a; i < b; ++i) {
            if (i + 8 < b) __builtin_prefetch(&x[o[i + 8] * p]);
            memcpy(&y[i * p], &x[o[i] * p], p * 8);
          }
        });
      for (auto& q : th) q.join();
      double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (rep) printf("threads %2d: %.1f ms  %.1f GB/s\n", T, s * 1e3, n * p * 8 / s / 1e9);
    }
  }
}
