// Throughput of the fp64 conversions the MLP epilogue uses (I2F.F64, F2F.F32.F64)
#include <cstdio>
__global__ void k_i2f(double* out, int iters) {
  long long c = threadIdx.x;
  double acc = 0;
  for (int i = 0; i < iters; i++) {
    acc += (double)(c + i) + (double)(c + 2 * i) + (double)(c + 3 * i) + (double)(c + 5 * i);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_f2f(float* out, int iters) {
  double x = threadIdx.x * 1e-3;
  float acc = 0;
  for (int i = 0; i < iters; i++) {
    acc += (float)(x + i) + (float)(x + 2.0 * i) + (float)(x + 3.0 * i) + (float)(x + 5.0 * i);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_dadd(double* out, int iters) {
  double x = threadIdx.x * 1e-3;
  double acc = 0;
  for (int i = 0; i < iters; i++) {
    acc += (x + i) + (x + 2.0 * i) + (x + 3.0 * i) + (x + 5.0 * i);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  double* d; float* f;
  cudaMalloc(&d, 148 * 8 * 256 * 8); cudaMalloc(&f, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000;
  const double n = 148.0 * 8 * 256 * iters * 4;
  float ms;
  k_i2f<<<148 * 8, 256>>>(d, 10);
  cudaEventRecord(e0); k_i2f<<<148 * 8, 256>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("I2F.F64 (+DADD): %.3f ms -> %.1f G/s (%.1f per clk per SM at 1.9 GHz)\n", ms, n / ms / 1e6, n / (ms * 1e-3) / 148 / 1.9e9);
  cudaEventRecord(e0); k_f2f<<<148 * 8, 256>>>(f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("F2F.F32.F64 (+DFMA): %.3f ms -> %.1f G/s (%.1f per clk per SM)\n", ms, n / ms / 1e6, n / (ms * 1e-3) / 148 / 1.9e9);
  cudaEventRecord(e0); k_dadd<<<148 * 8, 256>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("DFMA+DADD only: %.3f ms -> %.1f G/s (%.1f per clk per SM)\n", ms, n / ms / 1e6, n / (ms * 1e-3) / 148 / 1.9e9);
  return 0;
}
