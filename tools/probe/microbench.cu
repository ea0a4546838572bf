// Microbenchmarks for design decisions on B200 (sm_100a): FP64 add latency,
// POPC / FP64 / FP32 throughput, L2 random-gather bandwidth, H2D bandwidth.
// The last stdout line is a JSON object of the peaks (profiles/r2_microbench.json;
// bench.py's roofline.popc / roofline.l2_gather denominators).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dadd_chain(const double* in, double* out, int n) {
  double acc = 0.0;
  double x = in[threadIdx.x];
  for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, x * (double)i);  // dependent chain
  out[threadIdx.x] = acc;
}
__global__ void dadd_chain_pure(double x, double* out, int n) {
  double acc = 0.0;
  for (int i = 0; i < n; ++i) { acc = __dadd_rn(acc, x); }
  out[threadIdx.x] = acc;
}
__global__ void popc_tp(const uint32_t* in, uint32_t* out, int n) {
  uint32_t a = in[threadIdx.x], b = in[threadIdx.x + 1], c = in[threadIdx.x + 2], d = in[threadIdx.x + 3];
  uint32_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int i = 0; i < n; ++i) {
    s0 += __popc(a ^ i); s1 += __popc(b ^ i); s2 += __popc(c ^ i); s3 += __popc(d ^ i);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
__global__ void dfma_tp(double* out, int n) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  for (int i = 0; i < n; ++i) {
    a0 = __dadd_rn(a0, 1.0001); a1 = __dadd_rn(a1, 1.0001); a2 = __dadd_rn(a2, 1.0001); a3 = __dadd_rn(a3, 1.0001);
    a4 = __dadd_rn(a4, 1.0001); a5 = __dadd_rn(a5, 1.0001); a6 = __dadd_rn(a6, 1.0001); a7 = __dadd_rn(a7, 1.0001);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void ffma_tp(float* out, int n) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  for (int i = 0; i < n; ++i) {
    a0 = fmaf(a0, 1.0001f, 0.5f); a1 = fmaf(a1, 1.0001f, 0.5f); a2 = fmaf(a2, 1.0001f, 0.5f); a3 = fmaf(a3, 1.0001f, 0.5f);
    a4 = fmaf(a4, 1.0001f, 0.5f); a5 = fmaf(a5, 1.0001f, 0.5f); a6 = fmaf(a6, 1.0001f, 0.5f); a7 = fmaf(a7, 1.0001f, 0.5f);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
// random 16-byte gathers from a buffer of `words` uint4 entries (L2-resident when small)
__global__ void gather16(const uint4* __restrict__ buf, uint32_t mask, uint32_t* out, int iters) {
  uint32_t idx = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    idx = idx * 1664525u + 1013904223u;
    uint4 v = __ldcg(&buf[(idx >> 4) & mask]);
    acc += v.x ^ v.y ^ v.z ^ v.w;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
// warp-cooperative 512-byte row gathers (re-rank pattern)
__global__ void gather512(const float4* __restrict__ buf, uint32_t rows_mask, float* out, int iters) {
  int lane = threadIdx.x & 31;
  uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint32_t idx = w * 2654435761u;
  float acc = 0.f;
  for (int i = 0; i < iters; ++i) {
    idx = idx * 1664525u + 1013904223u;
    uint32_t r = (idx >> 8) & rows_mask;
    float4 v = __ldcg(&buf[(size_t)r * 32 + lane]);
    acc += v.x + v.y + v.z + v.w;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// 32-bit POPC throughput: 8 independent streams, one LOP3 + POPC + IADD each
__global__ void popc_pure(const uint32_t* in, uint32_t* out, int n) {
  uint32_t x[8], a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { x[k] = in[threadIdx.x + k]; a[k] = 0; }
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { a[k] += __popc(x[k] ^ (uint32_t)i); }
  }
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s sms %d l2 %d MB smemPerBlockOptin %zu clock %d kHz\n", p.name, p.multiProcessorCount,
         p.l2CacheSize >> 20, p.sharedMemPerBlockOptin, p.clockRate);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  double* dd; CK(cudaMalloc(&dd, 1 << 24));
  CK(cudaMemset(dd, 0, 1 << 24));
  int n = 1 << 20;
  dadd_chain_pure<<<1, 32>>>(1.5, dd, 1000); cudaDeviceSynchronize();
  cudaEventRecord(e0); dadd_chain_pure<<<1, 32>>>(1.5, dd, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("dadd chain: %.3f ms for %d dependent adds -> %.2f ns/add (%.2f cyc @ %.0f MHz)\n", ms, n, ms * 1e6 / n,
         ms * 1e6 / n * p.clockRate / 1e6, p.clockRate / 1e3);
  uint32_t* du; CK(cudaMalloc(&du, 64 << 20)); CK(cudaMemset(du, 1, 64 << 20));
  int blocks = p.multiProcessorCount * 8, threads = 256, it = 4096;
  double popc_pure_rate = 0, gather16_l2 = 0, gather16_hbm = 0, gather512_l2 = 0, dadd_rate = 0;
  popc_pure<<<blocks, threads>>>(du, du + 1024, 16); cudaDeviceSynchronize();
  cudaEventRecord(e0); popc_pure<<<blocks, threads>>>(du, du + 1024, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  popc_pure_rate = 8.0 * blocks * threads * it / (ms * 1e-3);
  printf("popc pure: %.3f ms, %.2f Tpopc/s -> %.1f per SM per clk\n", ms, popc_pure_rate / 1e12,
         popc_pure_rate / p.multiProcessorCount / (p.clockRate * 1e3));
  popc_tp<<<blocks, threads>>>(du, du + 1024, 16); cudaDeviceSynchronize();
  cudaEventRecord(e0); popc_tp<<<blocks, threads>>>(du, du + 1024, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double popcs = 4.0 * blocks * threads * it;
  printf("popc: %.3f ms, %.2f Tpopc/s -> %.1f per SM per clk\n", ms, popcs / ms / 1e9,
         popcs / (ms * 1e-3) / p.multiProcessorCount / (p.clockRate * 1e3));
  cudaEventRecord(e0); dfma_tp<<<blocks, threads>>>(dd, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double ops = 8.0 * blocks * threads * it;
  dadd_rate = ops / (ms * 1e-3);
  printf("dadd tp: %.3f ms, %.2f Tops/s -> %.1f per SM per clk\n", ms, ops / ms / 1e9,
         ops / (ms * 1e-3) / p.multiProcessorCount / (p.clockRate * 1e3));
  float* df; CK(cudaMalloc(&df, 64 << 20));
  cudaEventRecord(e0); ffma_tp<<<blocks, threads>>>(df, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("ffma tp: %.3f ms, %.2f Tfma/s -> %.1f per SM per clk\n", ms, ops / ms / 1e9,
         ops / (ms * 1e-3) / p.multiProcessorCount / (p.clockRate * 1e3));
  // L2 gathers: buffers of 4 MB (fits L2) and 1 GB (HBM)
  uint4* big; size_t bigbytes = size_t(1) << 30; CK(cudaMalloc(&big, bigbytes)); CK(cudaMemset(big, 3, bigbytes));
  for (int lg : {18, 20, 22, 24, 26}) {  // number of uint4 entries = 2^lg  (4 MB .. 1 GB)
    uint32_t mask = (1u << lg) - 1;
    int gi = 256;
    gather16<<<blocks, threads>>>(big, mask, du, 8); cudaDeviceSynchronize();
    cudaEventRecord(e0); gather16<<<blocks * 4, threads>>>(big, mask, du, gi); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double bytes = 16.0 * blocks * 4 * threads * gi;
    printf("gather16 over %zu MB: %.3f ms, %.1f GB/s (useful bytes)\n", (size_t(16) << lg) >> 20, ms, bytes / ms / 1e6);
    if (lg == 22) gather16_l2 = bytes / ms / 1e6;
    if (lg == 26) gather16_hbm = bytes / ms / 1e6;
  }
  for (int lg : {13, 15, 17, 21}) {  // rows of 512 B
    uint32_t mask = (1u << lg) - 1;
    int gi = 64;
    gather512<<<blocks, threads>>>((const float4*)big, mask, df, 8); cudaDeviceSynchronize();
    cudaEventRecord(e0); gather512<<<blocks * 4, threads>>>((const float4*)big, mask, df, gi); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double bytes = 512.0 * (blocks * 4 * threads / 32) * gi;
    printf("gather512 over %zu MB: %.3f ms, %.1f GB/s\n", (size_t(512) << lg) >> 20, ms, bytes / ms / 1e6);
    if (lg == 15) gather512_l2 = bytes / ms / 1e6;
  }
  // H2D pinned
  void* h; size_t hb = size_t(256) << 20; CK(cudaMallocHost(&h, hb)); memset(h, 1, hb);
  CK(cudaMemcpy(big, h, hb, cudaMemcpyHostToDevice));
  cudaEventRecord(e0); CK(cudaMemcpy(big, h, hb, cudaMemcpyHostToDevice)); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("H2D pinned 256MB: %.2f GB/s\n", hb / ms / 1e6);
  cudaEventRecord(e0); CK(cudaMemcpy(h, big, hb, cudaMemcpyDeviceToHost)); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("D2H pinned 256MB: %.2f GB/s\n", hb / ms / 1e6);
  std::vector<char> pg(hb, 1);
  cudaEventRecord(e0); CK(cudaMemcpy(big, pg.data(), hb, cudaMemcpyHostToDevice)); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("H2D pageable 256MB: %.2f GB/s\n", hb / ms / 1e6);
  printf("{\"popc32_per_s\": %.6g, \"dadd_per_s\": %.6g, \"gather16_l2_gbs\": %.6g, \"gather16_hbm_gbs\": %.6g, "
         "\"gather512_l2_gbs\": %.6g, \"sms\": %d, \"clock_khz\": %d}\n",
         popc_pure_rate, dadd_rate, gather16_l2, gather16_hbm, gather512_l2, p.multiProcessorCount, p.clockRate);
  return 0;
}
