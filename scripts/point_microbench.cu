// Latency of the grid-vertex position (vposition) as the MLP epilogue uses it
#include <cstdio>
#include "../paper_2409_13418_b200/csrc/odc_device.cuh"
#include "../paper_2409_13418_b200/csrc/odc_mlp.h"
using namespace odc;
__global__ void k(PointSrc src, long long* out, double* sink) {
  double p[3];
  long long t0 = clock64();
  vposition(src.grid, src.begin + blockIdx.x * blockDim.x + threadIdx.x, p);
  const float x0 = (float)(p[0] - 0.5), x1 = (float)(p[1] - 0.5), x2 = (float)(p[2] - 0.5);
  long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
int main() {
  PointSrc src{};
  GridP& g = src.grid;
  g.R = 512; g.S = 513; g.S2 = 513 * 513; g.S3 = g.S2 * 513; g.W = 17; g.nz = 513;
  for (int a = 0; a < 3; a++) { g.lo[a] = 0; g.h[a] = 1.0 / 512; }
  long long* o; double* sk;
  cudaMalloc(&o, 148 * 8); cudaMalloc(&sk, 148 * 256 * 8);
  k<<<148, 256>>>(src, o, sk);
  k<<<148, 256>>>(src, o, sk);
  long long h[148];
  cudaMemcpy(h, o, sizeof h, cudaMemcpyDeviceToHost);
  printf("vposition + 3 conversions: %lld cycles (block 0), %lld (block 100)\n", h[0], h[100]);
  return 0;
}
