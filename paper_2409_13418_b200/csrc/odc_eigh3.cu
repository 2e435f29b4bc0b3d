// Batched numpy.linalg.eigh for symmetric 3x3 matrices (odc_eigh3.cuh) on
// the device and on the host.  The QEF kernel (k_part_solve) inlines the
// same function; these entry points exist so the tests can pin the solver
// against numpy itself on arbitrary matrices (tests/test_eigh3.py,
// tests/test_gpu_eigh3.py).  Compiled with --fmad=false and host
// -ffp-contract=off: device and host execute the identical IEEE sequence.
#include "odc_eigh3.cuh"
#include "odc_kernels.h"

namespace odc {

__global__ void __launch_bounds__(128) k_eigh3_batch(const double* __restrict__ A, int64_t n, double* __restrict__ w,
                                                     double* __restrict__ V, int32_t* __restrict__ info) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double a[9], ww[3], vv[9];
  for (int k = 0; k < 9; k++) a[k] = A[9 * i + k];
  info[i] = odc_eigh3(a, ww, vv);
  for (int k = 0; k < 3; k++) w[3 * i + k] = ww[k];
  for (int k = 0; k < 9; k++) V[9 * i + k] = vv[k];
}

void launch_eigh3_batch(const double* A, int64_t n, double* w, double* V, int32_t* info, cudaStream_t s) {
  if (n > 0) k_eigh3_batch<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(A, n, w, V, info);
}

void eigh3_host_batch(const double* A, int64_t n, double* w, double* V, int32_t* info) {
  for (int64_t i = 0; i < n; i++) info[i] = odc_eigh3(A + 9 * i, w + 3 * i, V + 9 * i);
}

}  // namespace odc
