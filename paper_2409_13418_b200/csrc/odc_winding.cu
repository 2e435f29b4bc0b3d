// odc_winding.cu -- MeshWindingField on the device (occupancy from a triangle
// mesh by generalized winding numbers; /root/reference/pkg/src/occmesh/
// fields.py:281-386, _winding_batch and MeshWindingField).  SURVEY 8(f) item 4.
//
// raw(p) = sum over triangles of the signed solid angle
//          2 atan2(a . (b x c), |a||b||c| + (a.b)|c| + (b.c)|a| + (c.a)|b|)
// divided by 4 pi (Van Oosterom-Strackee), a, b, c = corners - p.  One thread
// per query walks all triangles.  The sum follows numpy's pairwise summation
// of omega.sum(axis=1) (blocks of 8 accumulators up to 128 terms, halving
// above), and every product/sum is in numpy's order (3-term einsum = (p0 + p2)
// + p1, norm = sqrt((x^2 + y^2) + z^2), no FMA), so the only difference from
// the reference is the device atan2 (<= 2 ulp per term).  A query that lies
// on a triangle (within 1e-12 of its plane, barycentric inside with 1e-12
// slack) is nudged by k * 1e-9 * scale / sqrt(3) along (1,1,1) on attempt k
// and retried, up to 8 attempts, like the reference's "perturb" mode.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "odc_device.cuh"
#include "odc_kernels.h"
#include "odc_mlp.h"

namespace odc {

namespace {
inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

struct W3 {
  double x, y, z;
};
__device__ __forceinline__ W3 ld3(const double* p, int64_t i) { return {p[3 * i], p[3 * i + 1], p[3 * i + 2]}; }
__device__ __forceinline__ W3 sub(W3 a, W3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ double ein(W3 a, W3 b) { return (a.x * b.x + a.z * b.z) + a.y * b.y; }
__device__ __forceinline__ double nrm(W3 a) { return sqrt((a.x * a.x + a.y * a.y) + a.z * a.z); }
__device__ __forceinline__ W3 crs(W3 a, W3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// signed solid angle of triangle t seen from p; sets hit when p lies on it
__device__ __forceinline__ double omega(const WindDev& w, W3 p, int64_t t, bool& hit) {
  const W3 A = ld3(w.ta, t), B = ld3(w.tb, t), C = ld3(w.tc, t);
  const W3 a = sub(A, p), b = sub(B, p), c = sub(C, p);
  const double la = nrm(a), lb = nrm(b), lc = nrm(c);
  const double num = ein(a, crs(b, c));
  const double den = ((la * lb * lc + ein(a, b) * lc) + ein(b, c) * la) + ein(c, a) * lb;
  if (w.ok[t] && fabs(ein(a, ld3(w.nhat, t))) <= 1e-12) {
    const W3 ap = sub(p, A);
    const double d20 = ein(ap, ld3(w.eab, t)), d21 = ein(ap, ld3(w.eac, t));
    const double v = (w.d11[t] * d20 - w.d01[t] * d21) / w.denb[t];
    const double u = (w.d00[t] * d21 - w.d01[t] * d20) / w.denb[t];
    if (v >= -1e-12 && u >= -1e-12 && v + u <= 1.0 + 1e-12) hit = true;
  }
  return 2.0 * atan2(num, den);
}

__device__ __forceinline__ void query_point(const PointSrc& s, int64_t i, double p[3]) {
  if (s.pts) {
    p[0] = s.pts[3 * i];
    p[1] = s.pts[3 * i + 1];
    p[2] = s.pts[3 * i + 2];
  } else {
    vposition(s.grid, s.begin + i, p);
  }
}

// one leaf of numpy's pairwise_sum (n <= 128): 8 accumulators, then the tail
__device__ double pw_leaf(const WindDev& w, W3 p, int64_t lo, int64_t n, bool& hit) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; i++) r += omega(w, p, lo + i, hit);
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; j++) r[j] = omega(w, p, lo + j, hit);
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] += omega(w, p, lo + i + j, hit);
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; i++) res += omega(w, p, lo + i, hit);
  return res;
}
__device__ __forceinline__ int64_t pw_half(int64_t n) {
  const int64_t n2 = n / 2;
  return n2 - n2 % 8;
}
// numpy pairwise_sum over omega(0 .. n): split in halves (rounded to a
// multiple of 8) down to leaves of <= 128 terms, combined left + right; the
// recursion is walked with an explicit stack (device stacks are small)
__device__ double pw_sum(const WindDev& w, W3 p, int64_t N, bool& hit) {
  int64_t lo_s[48], n_s[48];
  double left_s[48];
  bool right_s[48];
  int sp = 0;
  lo_s[0] = 0;
  n_s[0] = N;
  right_s[0] = false;
  for (;;) {
    const int64_t lo = lo_s[sp], n = n_s[sp];
    if (n > 128) {  // descend into the left half
      lo_s[sp + 1] = lo;
      n_s[sp + 1] = pw_half(n);
      right_s[sp + 1] = false;
      sp++;
      continue;
    }
    double v = pw_leaf(w, p, lo, n, hit);
    for (;;) {  // hand the value up
      if (sp == 0) return v;
      sp--;
      if (!right_s[sp]) {  // left half done: start the right half
        left_s[sp] = v;
        right_s[sp] = true;
        const int64_t n2 = pw_half(n_s[sp]);
        lo_s[sp + 1] = lo_s[sp] + n2;
        n_s[sp + 1] = n_s[sp] - n2;
        right_s[sp + 1] = false;
        sp++;
        break;
      }
      v = left_s[sp] + v;  // both halves done
    }
  }
}
}  // namespace

// per-triangle terms of _winding_batch's precomputation (fields.py:296-310)
__global__ void k_winding_prep(const double* __restrict__ v, const int64_t* __restrict__ t, int64_t nt, WindDev w) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nt) return;
  const W3 A = ld3(v, t[3 * i]), B = ld3(v, t[3 * i + 1]), C = ld3(v, t[3 * i + 2]);
  const W3 eab = sub(B, A), eac = sub(C, A);
  const W3 n = crs(eab, eac);
  const double len = nrm(n);
  const bool ok = len > 0;
  const W3 nh = ok ? W3{n.x / len, n.y / len, n.z / len} : W3{0.0, 0.0, 0.0};
  const double d00 = ein(eab, eab), d01 = ein(eab, eac), d11 = ein(eac, eac);
  double db = d00 * d11 - d01 * d01;
  if (fabs(db) < 1e-300) db = 1.0;
  const W3 out[6] = {A, B, C, nh, eab, eac};
  double* dst[6] = {w.ta, w.tb, w.tc, w.nhat, w.eab, w.eac};
  for (int k = 0; k < 6; k++) {
    dst[k][3 * i] = out[k].x;
    dst[k][3 * i + 1] = out[k].y;
    dst[k][3 * i + 2] = out[k].z;
  }
  w.ok[i] = ok;
  w.d00[i] = d00;
  w.d01[i] = d01;
  w.d11[i] = d11;
  w.denb[i] = db;
}
void launch_winding_prep(const double* v, const int64_t* t, int64_t nt, const WindDev& w, cudaStream_t s) {
  if (nt) k_winding_prep<<<grid_for(nt, 256), 256, 0, s>>>(v, t, nt, w);
}

__global__ void k_winding_eval(WindDev w, PointSrc src, int64_t n, uint8_t* __restrict__ labels,
                               double* __restrict__ raw, unsigned int* __restrict__ failed) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double q[3];
  query_point(src, i, q);
  W3 p{q[0], q[1], q[2]};
  double r = 0.0;
  bool done = false;
  for (int attempt = 0; attempt < 8 && !done; attempt++) {
    bool hit = false;
    const double s = pw_sum(w, p, w.nt, hit);
    if (!hit) {
      r = s / 12.566370614359172;  // FOUR_PI = 4.0 * math.pi
      done = true;
    } else {
      const double k = (double)(attempt + 1);
      p = {p.x + w.nudge * k, p.y + w.nudge * k, p.z + w.nudge * k};
    }
  }
  if (!done) {
    atomicOr(failed, 1u);
    r = 0.0;
  }
  if (labels) labels[i] = r > 0.5 ? 1 : 0;
  if (raw) raw[i] = r;
}
void winding_eval(const WindDev& w, const PointSrc& src, int64_t n, uint8_t* labels, double* raw,
                  unsigned int* failed, cudaStream_t s) {
  if (n) k_winding_eval<<<grid_for(n, 128), 128, 0, s>>>(w, src, n, labels, raw, failed);
}

}  // namespace odc
