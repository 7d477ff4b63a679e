// Which host-side CUDA runtime calls wait for a kernel running on ANOTHER
// non-blocking stream?  (Loopback-communicator design: a rank's host issue
// must never wait for another rank's spinning kernel.)
#include <cstdio>
#include <chrono>
#include <cuda_runtime.h>
__global__ void spin(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < ns);
}
static double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}
int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaFree(0);
  static char host[1 << 20];
  void* warm; cudaMalloc(&warm, 1 << 20); cudaFree(warm);
  const char* names[] = {"cudaMalloc 1MB", "cudaMalloc 256MB", "cudaMemcpy H2D pageable", "cudaMemset (sync)",
                         "cudaEventCreate", "cudaHostAlloc 1MB", "cudaFree", "cudaStreamCreate", "cudaMemcpyAsync H2D pageable on s2"};
  for (int test = 0; test < 9; ++test) {
    spin<<<1, 1, 0, s>>>(500ull * 1000 * 1000);  // 500 ms
    cudaDeviceSynchronize();  // (not in the measured part) restart:
    spin<<<1, 1, 0, s>>>(500ull * 1000 * 1000);
    auto t0 = std::chrono::steady_clock::now();
    void* p = nullptr; cudaEvent_t e; cudaStream_t s2;
    switch (test) {
      case 0: cudaMalloc(&p, 1 << 20); break;
      case 1: cudaMalloc(&p, 256 << 20); break;
      case 2: cudaMalloc(&p, 1 << 20); t0 = std::chrono::steady_clock::now(); cudaMemcpy(p, host, 1 << 20, cudaMemcpyHostToDevice); break;
      case 3: cudaMalloc(&p, 1 << 20); t0 = std::chrono::steady_clock::now(); cudaMemset(p, 0, 1 << 20); break;
      case 4: cudaEventCreate(&e); break;
      case 5: cudaHostAlloc(&p, 1 << 20, 0); break;
      case 6: cudaMalloc(&p, 1 << 20); t0 = std::chrono::steady_clock::now(); cudaFree(p); p = nullptr; break;
      case 7: cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking); break;
      case 8: cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking); cudaMalloc(&p, 1 << 20); t0 = std::chrono::steady_clock::now();
              cudaMemcpyAsync(p, host, 1 << 20, cudaMemcpyHostToDevice, s2); break;
    }
    printf("%-40s %8.2f ms (a 500 ms kernel runs on another non-blocking stream)\n", names[test], ms_since(t0));
    cudaDeviceSynchronize();
  }
  return 0;
}
