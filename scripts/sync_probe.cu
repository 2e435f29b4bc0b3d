// Host round-trip cost of a small device->host readback: kernel, 8-byte
// cudaMemcpyAsync, then (a) cudaStreamSynchronize or (b) a spin on
// cudaEventQuery.  nvcc -O2 -o /tmp/sync_probe scripts/sync_probe.cu
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>

__global__ void k_tiny(unsigned long long* p) {
  if (threadIdx.x == 0) p[0] += 1;
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  unsigned long long *d, *h;
  cudaMalloc(&d, 8);
  cudaMemset(d, 0, 8);
  cudaMallocHost(&h, 8);
  cudaEvent_t e;
  cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  const int n = 2000;
  for (int mode = 0; mode < 4; mode++) {
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; i++) {
      k_tiny<<<1, 32, 0, s>>>(d);
      if (mode == 3) {  // no readback: kernel launches only, one sync at the end
        continue;
      }
      cudaMemcpyAsync(h, d, 8, cudaMemcpyDeviceToHost, s);
      if (mode == 0) {
        cudaStreamSynchronize(s);
      } else if (mode == 1) {
        cudaEventRecord(e, s);
        while (cudaEventQuery(e) == cudaErrorNotReady) {
        }
      } else {
        cudaEventRecord(e, s);
        cudaEventSynchronize(e);
      }
    }
    cudaStreamSynchronize(s);
    auto t1 = std::chrono::steady_clock::now();
    const double us = std::chrono::duration<double, std::micro>(t1 - t0).count() / n;
    const char* names[] = {"stream sync", "event spin", "event sync", "launch only"};
    printf("%-12s %.2f us per kernel+readback\n", names[mode], us);
  }
  return 0;
}
