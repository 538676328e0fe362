// H2D staging micro-benchmark (run on the GPU box): DMA rate of an 8 MB chunk from
// a pinned stage, cold vs just written by the CPU, and chunk-size sensitivity.
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
using clk = std::chrono::steady_clock;
static double ms(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); }
int main() {
  const size_t B = 8u << 20;
  char* d; cudaMalloc(&d, 64u << 20);
  std::vector<char> src(64u << 20, 1);
  char *pin, *wc;
  cudaMallocHost(&pin, 64u << 20);
  cudaHostAlloc(&wc, 64u << 20, cudaHostAllocWriteCombined);
  memset(pin, 2, 64u << 20); memset(wc, 2, 64u << 20);
  cudaStream_t s; cudaStreamCreate(&s);
  for (int rep = 0; rep < 3; ++rep) {
    for (size_t b : {size_t(1) << 20, size_t(4) << 20, B, size_t(32) << 20}) {
      auto t0 = clk::now();
      cudaMemcpyAsync(d, pin, b, cudaMemcpyHostToDevice, s); cudaStreamSynchronize(s);
      auto t1 = clk::now();
      memcpy(pin, src.data(), b);
      auto t2 = clk::now();
      cudaMemcpyAsync(d, pin, b, cudaMemcpyHostToDevice, s); cudaStreamSynchronize(s);
      auto t3 = clk::now();
      cudaMemcpyAsync(d, wc, b, cudaMemcpyHostToDevice, s); cudaStreamSynchronize(s);
      auto t4 = clk::now();
      cudaMemcpyAsync(pin, d, b, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s);
      auto t5 = clk::now();
      cudaMemcpy(d, src.data(), b, cudaMemcpyHostToDevice);
      auto t6 = clk::now();
      printf("%5zu KB: pinned H2D %.3f ms (%.1f GB/s) | memcpy %.3f | H2D after write %.3f | WC H2D %.3f | D2H %.3f (%.1f GB/s) | pageable H2D %.3f\n",
             b >> 10, ms(t0, t1), b / ms(t0, t1) / 1e6, ms(t1, t2), ms(t2, t3), ms(t3, t4), ms(t4, t5), b / ms(t4, t5) / 1e6, ms(t5, t6));
    }
  }
  int dev; cudaGetDevice(&dev); int numa = -1;
  cudaDeviceGetAttribute(&numa, cudaDevAttrHostNumaId, dev);
  printf("host numa id of device: %d\n", numa);
}
