// Host-transfer micro-benchmark for the drop-in table copy (run on the GPU box):
// where does a pageable std::vector D2H of a C2-sized table spend its time?
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
using clk = std::chrono::steady_clock;
static double ms(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); }
int main() {
  const size_t N = 19628134;  // C2 items (int32) + offsets ~ 1M int64 (same order)
  int* d; cudaMalloc(&d, N * 4); cudaMemset(d, 1, N * 4); cudaDeviceSynchronize();
  for (int rep = 0; rep < 3; ++rep) {
    auto t0 = clk::now();
    { std::vector<int> v(N); auto t1 = clk::now();
      cudaMemcpy(v.data(), d, N * 4, cudaMemcpyDeviceToHost); auto t2 = clk::now();
      printf("A resize %.2f ms, pageable D2H %.2f ms\n", ms(t0, t1), ms(t1, t2)); }
    t0 = clk::now();
    { std::vector<int> v; v.reserve(N);
      uintptr_t p = ((uintptr_t)v.data() + (2u << 20) - 1) & ~(uintptr_t)((2u << 20) - 1);
      madvise((void*)p, N * 4 - (p - (uintptr_t)v.data()), MADV_HUGEPAGE);
      v.resize(N); auto t1 = clk::now();
      cudaMemcpy(v.data(), d, N * 4, cudaMemcpyDeviceToHost); auto t2 = clk::now();
      cudaHostRegister(v.data(), N * 4, cudaHostRegisterDefault); auto t3 = clk::now();
      cudaMemcpy(v.data(), d, N * 4, cudaMemcpyDeviceToHost); auto t4 = clk::now();
      cudaHostUnregister(v.data()); auto t5 = clk::now();
      printf("B hugepage resize %.2f, pageable D2H %.2f, register %.2f, pinned D2H %.2f, unregister %.2f\n",
             ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4), ms(t4, t5)); }
    // pinned staging + chunked copy into a reserved vector (insert: no zero-fill)
    static int* pin = nullptr; if (!pin) cudaMallocHost(&pin, 2 * (16u << 20));
    t0 = clk::now();
    { std::vector<int> v; v.reserve(N);
      uintptr_t p = ((uintptr_t)v.data() + (2u << 20) - 1) & ~(uintptr_t)((2u << 20) - 1);
      madvise((void*)p, N * 4 - (p - (uintptr_t)v.data()), MADV_HUGEPAGE);
      const size_t C = (16u << 20) / 4; cudaStream_t s; cudaStreamCreate(&s);
      cudaEvent_t ev[2]; cudaEventCreate(&ev[0]); cudaEventCreate(&ev[1]);
      size_t nch = (N + C - 1) / C;
      for (size_t c = 0; c < nch && c < 2; ++c) { size_t o = c * C, l = std::min(C, N - o);
        cudaMemcpyAsync(pin + (c & 1) * C, d + o, l * 4, cudaMemcpyDeviceToHost, s); cudaEventRecord(ev[c & 1], s); }
      for (size_t c = 0; c < nch; ++c) { size_t o = c * C, l = std::min(C, N - o);
        cudaEventSynchronize(ev[c & 1]);
        v.insert(v.end(), pin + (c & 1) * C, pin + (c & 1) * C + l);
        if (c + 2 < nch) { size_t o2 = (c + 2) * C, l2 = std::min(C, N - o2);
          cudaMemcpyAsync(pin + (c & 1) * C, d + o2, l2 * 4, cudaMemcpyDeviceToHost, s); cudaEventRecord(ev[c & 1], s); } }
      auto t1 = clk::now(); printf("C staged insert %.2f ms (size %zu)\n", ms(t0, t1), v.size());
      cudaStreamDestroy(s); }
    t0 = clk::now();
    { std::vector<int> v(N); auto t1 = clk::now();
      // 8-thread memcpy from pinned (full copy staged in one go)
      static int* big = nullptr; if (!big) cudaMallocHost(&big, N * 4);
      cudaMemcpy(big, d, N * 4, cudaMemcpyDeviceToHost); auto t2 = clk::now();
      std::vector<std::thread> th; for (int k = 0; k < 8; ++k) th.emplace_back([&, k] { size_t a = N * k / 8, b = N * (k + 1) / 8; memcpy(v.data() + a, big + a, (b - a) * 4); });
      for (auto& t : th) t.join(); auto t3 = clk::now();
      printf("D resize %.2f, pinned D2H %.2f, 8-thread memcpy %.2f\n", ms(t0, t1), ms(t1, t2), ms(t2, t3)); }
  }
  printf("threads %u\n", std::thread::hardware_concurrency());
}
