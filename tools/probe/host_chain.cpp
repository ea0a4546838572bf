// Host FP64 row-mean chain throughput (channel-split threads): how fast can
// the host reproduce engine.cpp:446-461 for a row of N images x 8194 desc?
// g++ -O3 -pthread tools/probe/host_chain.cpp -o /tmp/host_chain && /tmp/host_chain 400 8
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#ifndef CH
#define CH 16
#endif
int main(int argc, char** argv) {
  const int n_img = argc > 1 ? atoi(argv[1]) : 400, T = argc > 2 ? atoi(argv[2]) : 8;
  const size_t n = 8194;
  std::vector<float*> imgs(n_img);
  for (int i = 0; i < n_img; ++i) {
    imgs[i] = static_cast<float*>(aligned_alloc(64, n * 512));
    for (size_t k = 0; k < n * 128; ++k) imgs[i][k] = (float)((k * 2654435761u + i) % 1000) * 1e-3f;
  }
  for (int rep = 0; rep < 3; ++rep) {
    double acc[128] = {};
    const int per = 128 / T;
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        for (int c0 = t * per; c0 < (t + 1) * per; c0 += CH) {
          double a[CH] = {};
          for (int i = 0; i < n_img; ++i) {
            const float* d = imgs[i] + c0;
            for (size_t k = 0; k < n; ++k, d += 128)
#pragma GCC unroll 16
              for (int j = 0; j < CH; ++j) a[j] += (double)d[j];
          }
          for (int j = 0; j < CH; ++j) acc[c0 + j] = a[j];
        }
      });
    for (auto& x : th) x.join();
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("%d images, %d threads: %.2f ms  %.1f GB/s  (acc[0]=%g)\n", n_img, T, s * 1e3,
           n_img * n * 512.0 / s / 1e9, acc[0]);
  }
}
