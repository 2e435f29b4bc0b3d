// odc_voxel.cu -- VoxelField on the device (occupancy from a dense value
// grid by trilinear interpolation, zero outside; /root/reference/pkg/src/
// occmesh/fields.py:245-278).  Per query, in numpy's order and without FMA
// (this TU is built with --fmad=false), so raw values are bit-identical:
//   g = (p - origin) / spacing; inside = all(g >= 0) and all(g <= shape - 1)
//   i0 = clip(floor(g), 0, shape - 2); f = g - i0
//   c00 = v[i, j, k] (1 - fx) + v[i+1, j, k] fx  ... (x, then y, then z)
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "odc_device.cuh"
#include "odc_kernels.h"
#include "odc_mlp.h"

namespace odc {

namespace {
inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

__device__ __forceinline__ void vox_point(const PointSrc& s, int64_t i, double p[3]) {
  if (s.pts) {
    p[0] = s.pts[3 * i];
    p[1] = s.pts[3 * i + 1];
    p[2] = s.pts[3 * i + 2];
  } else {
    vposition(s.grid, s.begin + i, p);
  }
}
}  // namespace

__global__ void k_voxel_eval(VoxDev w, PointSrc src, int64_t n, uint8_t* __restrict__ labels,
                             double* __restrict__ raw) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double p[3];
  vox_point(src, i, p);
  const int64_t dim[3] = {w.nx, w.ny, w.nz};
  double g[3];
  bool inside = true;
#pragma unroll
  for (int a = 0; a < 3; a++) {
    g[a] = (p[a] - w.origin[a]) / w.spacing[a];
    inside &= g[a] >= 0.0 && g[a] <= (double)(dim[a] - 1);
  }
  double r = 0.0;
  if (inside) {
    int64_t i0[3];
    double f[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
      int64_t c = (int64_t)floor(g[a]);
      c = c < 0 ? 0 : (c > dim[a] - 2 ? dim[a] - 2 : c);
      i0[a] = c;
      f[a] = g[a] - (double)c;
    }
    auto V = [&](int64_t x, int64_t y, int64_t z) { return __ldg(w.values + (x * w.ny + y) * w.nz + z); };
    const int64_t x = i0[0], y = i0[1], z = i0[2];
    const double ux = 1.0 - f[0], uy = 1.0 - f[1], uz = 1.0 - f[2];
    const double c00 = V(x, y, z) * ux + V(x + 1, y, z) * f[0];
    const double c10 = V(x, y + 1, z) * ux + V(x + 1, y + 1, z) * f[0];
    const double c01 = V(x, y, z + 1) * ux + V(x + 1, y, z + 1) * f[0];
    const double c11 = V(x, y + 1, z + 1) * ux + V(x + 1, y + 1, z + 1) * f[0];
    const double c0 = c00 * uy + c10 * f[1];
    const double c1 = c01 * uy + c11 * f[1];
    r = c0 * uz + c1 * f[2];
  }
  if (labels) labels[i] = r > 0.5 ? 1 : 0;
  if (raw) raw[i] = r;
}

void voxel_eval(const VoxDev& w, const PointSrc& src, int64_t n, uint8_t* labels, double* raw, cudaStream_t s) {
  if (n) k_voxel_eval<<<grid_for(n, 256), 256, 0, s>>>(w, src, n, labels, raw);
}

}  // namespace odc
