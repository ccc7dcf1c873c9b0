// D3Q19 lattice, block layouts and node metadata encoding, as compile-time
// functions so every per-direction quantity folds to an immediate once the
// direction loop is unrolled.
//
// Direction order, vectors and weights: reference lattice.py:22-59.
// Layouts: L_XYZ / L_YXZ / L_zigzagNE from layout.py:45-58, plus L_ZXY
// (z fastest) used by the B200 table for the four XY diagonals so that every
// 32-byte sector of a block is consumed by exactly one destination tile
// (304 read sectors per tile = the minimum, vs 344 for the
// paper's table).
#pragma once
#include <cstdint>

namespace tlbm {

constexpr int Q = 19;

__host__ __device__ constexpr int ex(int q) {
    return (q == 1 || q == 7 || q == 9 || q == 15 || q == 16) ? 1
         : (q == 3 || q == 8 || q == 10 || q == 17 || q == 18) ? -1 : 0;
}
__host__ __device__ constexpr int ey(int q) {
    return (q == 2 || q == 7 || q == 8 || q == 11 || q == 12) ? 1
         : (q == 4 || q == 9 || q == 10 || q == 13 || q == 14) ? -1 : 0;
}
__host__ __device__ constexpr int ez(int q) {
    return (q == 5 || q == 11 || q == 13 || q == 15 || q == 17) ? 1
         : (q == 6 || q == 12 || q == 14 || q == 16 || q == 18) ? -1 : 0;
}
__host__ __device__ constexpr int e_axis(int q, int a) {
    return a == 0 ? ex(q) : (a == 1 ? ey(q) : ez(q));
}
__host__ __device__ constexpr int opp(int q) {
    // lattice.py:56-59: axis pairs (E,W) (N,S) (T,B); diagonal pairs sum to
    // 17 (NE..SW), 25 (NT..SB), 33 (ET..WB)
    return q == 0 ? 0
         : q == 1 ? 3 : q == 3 ? 1 : q == 2 ? 4 : q == 4 ? 2
         : q == 5 ? 6 : q == 6 ? 5
         : q <= 10 ? 17 - q : (q <= 14 ? 25 - q : 33 - q);
}
__host__ __device__ constexpr double weight(int q) {
    return q == 0 ? 1.0 / 3.0 : (q <= 6 ? 1.0 / 18.0 : 1.0 / 36.0);
}

// ---- layouts -------------------------------------------------------------
enum Kind : int { K_XYZ = 0, K_YXZ = 1, K_ZIGZAG = 2, K_ZXY = 3 };
enum Table : int { T_XYZ = 0, T_OPTIMIZED = 1, T_B200 = 2 };

__host__ __device__ constexpr int layout_slot(int kind, int x, int y, int z) {
    return kind == K_XYZ ? x + 4 * y + 16 * z
         : kind == K_YXZ ? y + 4 * x + 16 * z
         : kind == K_ZXY ? z + 4 * x + 16 * y
         : 2 * (x + 3 * y + ((x + 1) & 4) * (3 - y)) + (z & 1) + 16 * (z & 2);
}

// layout.py:76-105 for T_OPTIMIZED; T_B200 differs only in NW/SW/NE/SE -> ZXY
__host__ __device__ constexpr int kind_of(int table, int q) {
    return table == T_XYZ ? K_XYZ
         : (ex(q) == 0) ? K_XYZ
         : (table == T_B200 && ey(q) != 0) ? K_ZXY
         : (table == T_OPTIMIZED && (q == 7 || q == 9)) ? K_ZIGZAG
         : K_YXZ;
}

// compact storage (compact.cu, step_compact.cuh) keeps every block in the
// canonical XYZ slot order, so a node's rank is one number for all 19 blocks
__host__ __device__ constexpr bool compact_table_ok(int table) { return table == T_XYZ; }

template <int TABLE>
__device__ __forceinline__ int slot_of(int q, int x, int y, int z) {
    return layout_slot(kind_of(TABLE, q), x, y, z);
}

// ---- node metadata word (one uint32 per tile slot) ------------------------
// bit 0       node is non-solid and inside the domain (it is updated)
// bits 1..18  bit q: the pull source n - e_q is non-solid and in the domain
//             (after periodic wrap); clear -> halfway bounce-back fill
// bits 19..21 node type (geometry.py NodeType)
// bits 22..24 Zou-He face id 2*axis + (0 low | 1 high) for inlet/outlet nodes
constexpr uint32_t META_ACTIVE = 1u;
__host__ __device__ constexpr int meta_type(uint32_t m) { return (m >> 19) & 7; }
__host__ __device__ constexpr int meta_face(uint32_t m) { return (m >> 22) & 7; }

enum NodeTag : int { SOLID = 0, FLUID = 1, BB_WALL = 2, INLET = 3, OUTLET = 4 };

// neighbour-table column of tile delta (dx, dy, dz) in {-1,0,1}^3; the same
// order as itertools.product((-1, 0, 1), repeat=3)
__host__ __device__ constexpr int delta_index(int dx, int dy, int dz) {
    return 9 * (dx + 1) + 3 * (dy + 1) + (dz + 1);
}
constexpr int NBR = 27;

}  // namespace tlbm
