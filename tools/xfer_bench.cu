// Host<->device transfer options for the e2e path (not part of the product).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
using clk = std::chrono::steady_clock;
static double ms(clk::time_point a) { return std::chrono::duration<double, std::milli>(clk::now() - a).count(); }
int main() {
  for (size_t bytes : {16ull << 20, 100ull << 20}) {
    void* d; cudaMalloc(&d, bytes);
    std::vector<char> pageable(bytes, 1);
    void* pinned; cudaMallocHost(&pinned, bytes);
    cudaMemcpy(d, pinned, bytes, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 2; ++rep) {
      auto t = clk::now(); cudaMemcpy(pageable.data(), d, bytes, cudaMemcpyDeviceToHost); double a = ms(t);
      t = clk::now(); cudaMemcpy(pinned, d, bytes, cudaMemcpyDeviceToHost); double b = ms(t);
      t = clk::now(); std::memcpy(pageable.data(), pinned, bytes); double c = ms(t);
      t = clk::now();
      {
        int T = 8; std::vector<std::thread> th;
        for (int i = 0; i < T; ++i) th.emplace_back([&, i] { size_t lo = bytes * i / T, hi = bytes * (i + 1) / T; std::memcpy(pageable.data() + lo, (char*)pinned + lo, hi - lo); });
        for (auto& x : th) x.join();
      }
      double c8 = ms(t);
      t = clk::now(); cudaHostRegister(pageable.data(), bytes, 0); double reg = ms(t);
      t = clk::now(); cudaMemcpy(pageable.data(), d, bytes, cudaMemcpyDeviceToHost); double e = ms(t);
      t = clk::now(); cudaHostUnregister(pageable.data()); double unreg = ms(t);
      t = clk::now(); cudaMemcpy(d, pageable.data(), bytes, cudaMemcpyHostToDevice); double h2dp = ms(t);
      t = clk::now(); cudaMemcpy(d, pinned, bytes, cudaMemcpyHostToDevice); double h2dpin = ms(t);
      printf("%zu MB: D2H pageable %.3f | D2H pinned %.3f + memcpy %.3f (8thr %.3f) | register %.3f D2H %.3f unregister %.3f | H2D pageable %.3f pinned %.3f ms\n",
             bytes >> 20, a, b, c, c8, reg, e, unreg, h2dp, h2dpin);
    }
  }
}
