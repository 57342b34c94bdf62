// Host memory bandwidth of the GPU box (the roofline of the host side of an
// e2e call once the link is no longer the bound): T threads each reading,
// writing, or copying its own slice of a 2 GB buffer, best of 5.
//
//   g++ -O3 -march=native -pthread -o host_bw tools/host_bw.cpp && ./host_bw
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <chrono>
#include <thread>
#include <vector>

int main() {
  const size_t n = (size_t)1 << 28;                       // 2 GB of uint64
  std::vector<uint64_t> a(n, 1), b(n, 2);
  unsigned hw = std::thread::hardware_concurrency();
  volatile uint64_t sink = 0;
  for (unsigned T : {1u, 4u, 8u, hw}) {
    for (int kind = 0; kind < 3; ++kind) {
      double best = 1e30;
      for (int rep = 0; rep < 5; ++rep) {
        std::vector<std::thread> th;
        std::vector<uint64_t> part(T, 0);
        auto t0 = std::chrono::steady_clock::now();
        for (unsigned k = 0; k < T; ++k)
          th.emplace_back([&, k] {
            const size_t lo = n * k / T, hi = n * (k + 1) / T;
            if (kind == 0) {
              uint64_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
              for (size_t i = lo; i + 4 <= hi; i += 4) { s0 ^= a[i]; s1 ^= a[i + 1]; s2 ^= a[i + 2]; s3 ^= a[i + 3]; }
              part[k] = s0 ^ s1 ^ s2 ^ s3;
            } else if (kind == 1) {
              memset(&b[lo], k, (hi - lo) * 8);
            } else {
              memcpy(&b[lo], &a[lo], (hi - lo) * 8);
            }
          });
        for (auto& t : th) t.join();
        double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (uint64_t p : part) sink = sink ^ p;
        if (s < best) best = s;
      }
      const double bytes = (kind == 2 ? 2.0 : 1.0) * n * 8;
      printf("threads %2u  %-6s %6.1f GB/s%s\n", T, kind == 0 ? "read" : kind == 1 ? "write" : "copy",
             bytes / best / 1e9, kind == 2 ? " (read + write)" : "");
    }
  }
  return (int)(sink & 0);
}
