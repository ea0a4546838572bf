// H2D of N separate pinned images (4.2 MB each) into N separate device
// buffers, one copy per image, vs one contiguous copy of the same bytes and
// copies of two images at a time.  nvcc -O2 tools/probe/h2d_sizes.cu -o /tmp/h2ds
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <vector>
int main() {
  const int n = 100;
  const size_t b = 8194ull * 512;
  std::vector<void*> h(n), d(n);
  for (int i = 0; i < n; ++i) {
    cudaMallocHost(&h[i], b);
    cudaMalloc(&d[i], b);
  }
  void *hc, *dc;
  cudaMallocHost(&hc, b * n);
  cudaMalloc(&dc, b * n);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time = [&](auto&& f, const char* what) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0, s);
      f();
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    printf("%-28s %7.3f ms  %6.1f GB/s  (%s)\n", what, best, n * b / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  time([&] { for (int i = 0; i < n; ++i) cudaMemcpyAsync(d[i], h[i], b, cudaMemcpyHostToDevice, s); }, "per-image cudaMemcpyAsync");
  time([&] { cudaMemcpyAsync(dc, hc, b * n, cudaMemcpyHostToDevice, s); }, "one contiguous copy");
  time([&] { for (int i = 0; i < n; i += 2) cudaMemcpyAsync((char*)dc + i * b, (char*)hc + i * b, 2 * b, cudaMemcpyHostToDevice, s); }, "pairs of images (8.4 MB)");
}
