// Host FP64 chain (channel-split threads, AVX-512 when available) while the
// copy engine streams other pinned images to the GPU: does the host keep up?
// nvcc -O3 -Xcompiler -mavx512f,-pthread tools/probe/host_chain_dma.cu -o /tmp/hcd && /tmp/hcd
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>
#include <type_traits>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
  const size_t n = 8194, img_b = n * 512;
  const int n_chain = 200, n_dma = 400;
  std::vector<float*> imgs(n_chain + n_dma);
  for (auto& p : imgs) {
    cudaMallocHost(&p, img_b);
    for (size_t k = 0; k < n * 128; ++k) p[k] = (float)(k % 977) * 1e-3f;
  }
  float* d;
  cudaMalloc(&d, img_b * n_dma);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int mode = 0; mode < 3; ++mode) {  // 0: chain alone, 1: DMA alone, 2: both
    for (int T : {8, 16}) {
      if (mode == 1 && T == 16) continue;
      const double t0 = now();
      if (mode) for (int i = 0; i < n_dma; ++i) cudaMemcpyAsync(d + (size_t)i * n * 128, imgs[n_chain + i], img_b, cudaMemcpyHostToDevice, s);
      double tc = 0;
      if (mode != 1) {
        std::vector<std::thread> th;
        double acc[128];
        const int per = 128 / T;
        auto run = [&](auto width, int t) {
          constexpr int W = decltype(width)::value;
          const int c0 = t * W;
          double a[W] = {};
          for (int i = 0; i < n_chain; ++i) {
            const float* x = imgs[i] + c0;
            for (size_t k = 0; k < n; ++k, x += 128)
#pragma GCC unroll 16
              for (int j = 0; j < W; ++j) a[j] += (double)x[j];
          }
          for (int j = 0; j < W; ++j) acc[c0 + j] = a[j];
        };
        for (int t = 0; t < T; ++t)
          th.emplace_back([&, t] {
            if (per == 16) run(std::integral_constant<int, 16>{}, t);
            else run(std::integral_constant<int, 8>{}, t);
          });
        for (auto& x : th) x.join();
        tc = now() - t0;
      }
      cudaStreamSynchronize(s);
      const double td = now() - t0;
      printf("mode %d T=%2d: chain %.1f ms (%.1f GB/s)  dma+chain %.1f ms (dma %.1f GB/s)\n", mode, T, tc * 1e3,
             tc > 0 ? n_chain * img_b / tc / 1e9 : 0.0, td * 1e3, mode ? n_dma * img_b / td / 1e9 : 0.0);
    }
  }
}
