#include <cstdio>
__global__ void k(double* out, int iters, double a) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; i++) {
    x0 = x0 * a + 1e-9; x1 = x1 * a + 1e-9; x2 = x2 * a + 1e-9; x3 = x3 * a + 1e-9;
    x4 = x4 * a + 1e-9; x5 = x5 * a + 1e-9; x6 = x6 * a + 1e-9; x7 = x7 * a + 1e-9;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void kf(float* out, int iters, float a) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; i++) {
    x0 = x0 * a + 1e-9f; x1 = x1 * a + 1e-9f; x2 = x2 * a + 1e-9f; x3 = x3 * a + 1e-9f;
    x4 = x4 * a + 1e-9f; x5 = x5 * a + 1e-9f; x6 = x6 * a + 1e-9f; x7 = x7 * a + 1e-9f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  double* d; float* f;
  cudaMalloc(&d, 148 * 8 * 256 * 8); cudaMalloc(&f, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  k<<<148 * 8, 256>>>(d, 10, 0.999);
  cudaEventRecord(e0); k<<<148 * 8, 256>>>(d, iters, 0.999); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = 148.0 * 8 * 256 * iters * 8 * 2;
  printf("fp64 FMA: %.3f ms -> %.2f TFLOP/s\n", ms, ops / ms / 1e9);
  cudaEventRecord(e0); kf<<<148 * 8, 256>>>(f, iters, 0.999f); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("fp32 FMA: %.3f ms -> %.2f TFLOP/s\n", ms, ops / ms / 1e9);
  return 0;
}
