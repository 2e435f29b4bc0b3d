// odc_meshio.cpp -- mesh output formats of the extraction path
// (/root/reference/pkg/src/occmesh/meshio.py:22-98), host side.
//
// OBJ: "v x y z" lines with every coordinate printed as %.17g (Python's
// f"{x:.17g}" and glibc's printf are both correctly rounded and share the
// 'g' rules, so the bytes are identical), then "f i j k" with 1-based
// indices; lines joined by '\n' plus a final '\n' when the mesh is not
// empty (meshio.py:22-28).  Formatting 10^6-10^7 numbers is the cost, so rows
// are formatted in parallel chunks and written in order.
//
// PLY: the binary little-endian subset of meshio.py:79-98: ASCII header,
// float32 xyz per vertex (round-to-nearest from f64, numpy astype("<f4")),
// then per face one uchar 3 and three int32 (astype("<i4")).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/odc.h"

namespace {

// unsigned decimal, returns the end pointer
inline char* put_u64(char* p, uint64_t x) {
  char tmp[24];
  int n = 0;
  do {
    tmp[n++] = (char)('0' + x % 10);
    x /= 10;
  } while (x);
  while (n) *p++ = tmp[--n];
  return p;
}
inline char* put_i64(char* p, int64_t x) {
  if (x < 0) {
    *p++ = '-';
    return put_u64(p, (uint64_t)(-(x + 1)) + 1);
  }
  return put_u64(p, (uint64_t)x);
}

template <class F>
void parallel_chunks(int64_t n, int64_t chunk, F&& fn) {
  const int64_t nchunks = (n + chunk - 1) / chunk;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int64_t nthr = std::min<int64_t>({(int64_t)16, (int64_t)hw, nchunks});
  if (nthr <= 1) {
    for (int64_t c = 0; c < nchunks; c++) fn(c);
    return;
  }
  std::vector<std::thread> pool;
  for (int64_t t = 0; t < nthr; t++)
    pool.emplace_back([&, t]() {
      for (int64_t c = t; c < nchunks; c += nthr) fn(c);
    });
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" int odc_export_obj(const char* path, const double* v, int64_t nv, const int64_t* t, int64_t nt) {
  if (!path || nv < 0 || nt < 0 || (nv && !v) || (nt && !t)) return ODC_E_ARG;
  constexpr int64_t kRows = 1 << 15;
  const int64_t vchunks = (nv + kRows - 1) / kRows, tchunks = (nt + kRows - 1) / kRows;
  std::vector<std::string> parts(vchunks + tchunks);
  parallel_chunks(vchunks + tchunks, 1, [&](int64_t c) {
    std::string& s = parts[c];
    if (c < vchunks) {
      const int64_t r0 = c * kRows, r1 = std::min(nv, r0 + kRows);
      s.resize((size_t)(r1 - r0) * 80);
      char* p = &s[0];
      for (int64_t r = r0; r < r1; r++) {
        const double* x = v + 3 * r;
        p += std::snprintf(p, 80, "v %.17g %.17g %.17g\n", x[0], x[1], x[2]);
      }
      s.resize(p - &s[0]);
    } else {
      const int64_t r0 = (c - vchunks) * kRows, r1 = std::min(nt, r0 + kRows);
      s.resize((size_t)(r1 - r0) * 72);
      char* p = &s[0];
      for (int64_t r = r0; r < r1; r++) {
        const int64_t* f = t + 3 * r;
        *p++ = 'f';
        for (int k = 0; k < 3; k++) {
          *p++ = ' ';
          p = put_i64(p, f[k] + 1);
        }
        *p++ = '\n';
      }
      s.resize(p - &s[0]);
    }
  });
  FILE* fh = std::fopen(path, "wb");
  if (!fh) return ODC_E_ARG;
  bool ok = true;
  for (const std::string& s : parts)
    if (!s.empty() && std::fwrite(s.data(), 1, s.size(), fh) != s.size()) ok = false;
  if (std::fclose(fh) != 0) ok = false;
  return ok ? ODC_OK : ODC_E_ARG;
}

extern "C" int odc_export_ply(const char* path, const double* v, int64_t nv, const int64_t* t, int64_t nt) {
  if (!path || nv < 0 || nt < 0 || (nv && !v) || (nt && !t)) return ODC_E_ARG;
  std::string header = "ply\nformat binary_little_endian 1.0\nelement vertex ";
  header += std::to_string(nv);
  header += "\nproperty float x\nproperty float y\nproperty float z\nelement face ";
  header += std::to_string(nt);
  header += "\nproperty list uchar int vertex_indices\nend_header\n";
  std::vector<float> vf((size_t)nv * 3);
  parallel_chunks(nv * 3, 1 << 20, [&](int64_t c) {
    const int64_t i0 = c << 20, i1 = std::min(nv * 3, i0 + (1 << 20));
    for (int64_t i = i0; i < i1; i++) vf[i] = (float)v[i];
  });
  std::vector<unsigned char> body((size_t)nt * 13);
  parallel_chunks(nt, 1 << 18, [&](int64_t c) {
    const int64_t r0 = c << 18, r1 = std::min(nt, r0 + (1 << 18));
    for (int64_t r = r0; r < r1; r++) {
      unsigned char* q = &body[(size_t)r * 13];
      q[0] = 3;
      for (int k = 0; k < 3; k++) {
        const uint32_t x = (uint32_t)(int32_t)t[3 * r + k];  // astype("<i4") wraps like a C cast
        q[1 + 4 * k] = (unsigned char)(x & 0xff);
        q[2 + 4 * k] = (unsigned char)((x >> 8) & 0xff);
        q[3 + 4 * k] = (unsigned char)((x >> 16) & 0xff);
        q[4 + 4 * k] = (unsigned char)(x >> 24);
      }
    }
  });
  FILE* fh = std::fopen(path, "wb");
  if (!fh) return ODC_E_ARG;
  bool ok = std::fwrite(header.data(), 1, header.size(), fh) == header.size();
  static_assert(sizeof(float) == 4, "float32");
  if (nv) {  // x86-64 / aarch64 hosts are little-endian, like "<f4"
    ok = ok && std::fwrite(vf.data(), 4, vf.size(), fh) == vf.size();
  }
  if (nt) ok = ok && std::fwrite(body.data(), 1, body.size(), fh) == body.size();
  if (std::fclose(fh) != 0) ok = false;
  return ok ? ODC_OK : ODC_E_ARG;
}
