// odc_tables.cpp -- host construction of the per-cell cycle table.
//
// For every (8-bit corner configuration, 6-bit face-centre mask) this runs the
// face pairing rule (_pair_rule, dualize.py:37-48; 2-crossing faces pair their
// two crossing edges, dualize.py:76-78) and trace_cycles (dualize.py:132-165)
// with local edge ids in key order and local instance codes (face in key
// order, slot) in global-instance order.
#include "odc_tables.h"

#include <algorithm>
#include <cstring>
#include <vector>

namespace odc {

namespace {

int local_edge(int corner, int axis) {
  for (int e = 0; e < 12; e++)
    if (kLE_CORNER[e] == corner && kLE_AXIS[e] == axis) return e;
  return -1;
}

// Self-check that the hard-coded key orders are what the global keys give.
bool check_orders() {
  const long S = 7, S2 = S * S;
  auto off = [&](int c) { return (long)(c & 1) + ((c >> 1) & 1) * S + ((c >> 2) & 1) * S2; };
  std::vector<std::pair<long, int>> ek;
  for (int c = 0; c < 8; c++)
    for (int a = 0; a < 3; a++)
      if (!((c >> a) & 1)) ek.push_back({off(c) * 3 + a, c * 3 + a});
  std::sort(ek.begin(), ek.end());
  if (ek.size() != 12) return false;
  for (int e = 0; e < 12; e++)
    if (ek[e].second != kLE_CORNER[e] * 3 + kLE_AXIS[e]) return false;
  std::vector<std::pair<long, int>> fk;
  for (int a = 0; a < 3; a++)
    for (int side = 0; side < 2; side++) {
      int c = side << a;
      fk.push_back({off(c) * 3 + a, c * 3 + a});
    }
  std::sort(fk.begin(), fk.end());
  for (int f = 0; f < 6; f++)
    if (fk[f].second != kLF_CORNER[f] * 3 + kLF_NORMAL[f]) return false;
  return true;
}

}  // namespace

int build_cell_table(CellTabEntry* table) {
  if (!check_orders()) return -1;
  for (int cfg = 0; cfg < 256; cfg++) {
    int lab[8];
    for (int i = 0; i < 8; i++) lab[i] = (cfg >> i) & 1;
    bool crossing[12];
    for (int e = 0; e < 12; e++) {
      int c0 = kLE_CORNER[e], c1 = c0 | (1 << kLE_AXIS[e]);
      crossing[e] = lab[c0] != lab[c1];
    }
    for (int cm = 0; cm < 64; cm++) {
      CellTabEntry& T = table[cfg * 64 + cm];
      std::memset(&T, 0, sizeof T);
      // joins[e] = list of (instance code, other edge)
      int jn[12] = {0}, jinst[12][4], joth[12][4];
      for (int f = 0; f < 6; f++) {
        int n = kLF_NORMAL[f], b = (n + 1) % 3, c = (n + 2) % 3;
        int w0 = kLF_CORNER[f], w1 = w0 | (1 << b), w3 = w0 | (1 << c);
        int ed[4] = {local_edge(w0, b), local_edge(w1, c), local_edge(w3, b), local_edge(w0, c)};
        int nc = 0, sel[4];
        for (int j = 0; j < 4; j++)
          if (crossing[ed[j]]) sel[nc++] = ed[j];
        int pairs[2][2], np = 0;
        if (nc == 2) {
          pairs[0][0] = sel[0]; pairs[0][1] = sel[1]; np = 1;
        } else if (nc == 4) {
          int centre = (cm >> f) & 1;
          if (centre == lab[w0]) {
            pairs[0][0] = ed[0]; pairs[0][1] = ed[1]; pairs[1][0] = ed[2]; pairs[1][1] = ed[3];
          } else {
            pairs[0][0] = ed[3]; pairs[0][1] = ed[0]; pairs[1][0] = ed[1]; pairs[1][1] = ed[2];
          }
          np = 2;
        } else if (nc != 0) {
          return -2;  // odd crossing count is impossible
        }
        for (int s = 0; s < np; s++) {
          int a = std::min(pairs[s][0], pairs[s][1]), bb = std::max(pairs[s][0], pairs[s][1]);
          int code = f * 2 + s;
          jinst[a][jn[a]] = code; joth[a][jn[a]] = bb; jn[a]++;
          jinst[bb][jn[bb]] = code; joth[bb][jn[bb]] = a; jn[bb]++;
        }
      }
      bool visited[12] = {false};
      int slot = 0, ncyc = 0;
      for (int start = 0; start < 12; start++) {
        if (!crossing[start] || visited[start]) continue;
        if (jn[start] != 2) return -3;
        int m = (jinst[start][1] < jinst[start][0] ||
                 (jinst[start][1] == jinst[start][0] && joth[start][1] < joth[start][0])) ? 1 : 0;
        int inst = jinst[start][m], nxt = joth[start][m], prev = inst;
        visited[start] = true;
        int len = 0;
        T.edges |= (uint64_t)start << (4 * slot);
        T.insts |= (uint64_t)inst << (4 * slot);
        T.cyc_of_edge |= (uint32_t)ncyc << (2 * start);
        slot++; len++;
        while (nxt != start) {
          if (visited[nxt] || jn[nxt] != 2) return -4;
          visited[nxt] = true;
          int pick = (jinst[nxt][0] != prev) ? 0 : 1;
          if (jinst[nxt][1 - pick] != prev) return -5;
          T.edges |= (uint64_t)nxt << (4 * slot);
          T.cyc_of_edge |= (uint32_t)ncyc << (2 * nxt);
          inst = jinst[nxt][pick];
          T.insts |= (uint64_t)inst << (4 * slot);
          slot++; len++;
          prev = inst;
          nxt = joth[nxt][pick];
        }
        T.lens |= (uint16_t)(len << (4 * ncyc));
        ncyc++;
      }
      T.ncyc = (uint8_t)ncyc;
      T.nedge = (uint8_t)slot;
    }
  }
  return 0;
}

}  // namespace odc
