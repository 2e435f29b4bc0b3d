// odc_tables.h -- local cell topology in key order and the per-cell cycle
// table that replaces partition_cells' Python loop (dualize.py:194-238).
//
// Within one cell the global edge-key order and face-key order are the same
// for every cell (S >= 3), so trace_cycles (dualize.py:132-165) -- start at
// the smallest unvisited edge key, first join = min(instance id, other edge),
// then follow the other join -- depends only on the 8 corner labels and the
// face-centre labels of the cell's 4-crossing faces.  The table maps
// (corner config, centre mask) -> cycles, built on the host by literally
// tracing with local ids in key order.
#pragma once
#include <cstdint>

namespace odc {

// local edges in ascending global key order: (corner, axis); corner bit i ->
// (i&1, i>>1&1, i>>2&1); key = (base + off(corner))*3 + axis
constexpr int kLE_CORNER[12] = {0, 0, 0, 1, 1, 2, 2, 3, 4, 4, 5, 6};
constexpr int kLE_AXIS[12] = {0, 1, 2, 1, 2, 0, 2, 2, 0, 1, 1, 0};
// local faces in ascending global key order: (corner, normal axis)
constexpr int kLF_CORNER[6] = {0, 0, 0, 1, 2, 4};
constexpr int kLF_NORMAL[6] = {0, 1, 2, 0, 1, 2};

struct CellTabEntry {
  uint64_t edges;        // 4 bits per slot: local edge ids in cycle order, cycles concatenated
  uint64_t insts;        // 4 bits per slot: local instance code (face*2 + slot); instance j joins edge j and j+1
  uint32_t cyc_of_edge;  // 2 bits per local edge: cycle index
  uint16_t lens;         // 4 bits per cycle
  uint8_t ncyc;
  uint8_t nedge;
};
static_assert(sizeof(CellTabEntry) == 24, "table entry layout");

constexpr int kTableSize = 256 * 64;

// Host: fill table[kTableSize]; returns 0 on success.
int build_cell_table(CellTabEntry* table);

}  // namespace odc
