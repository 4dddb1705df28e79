// Reusable pieces of the TMA -> smem -> DMMA tile pipeline shared by the GEMM
// (gemm.cu) and the fused triangular solve (trsm.cu).
//
// smem stage layout for a BM x BN output tile and BK = 16:
//   A: BM/16 boxes of 16 (m) x 16 (k) doubles, SWIZZLE_128B, 2 KB each
//      (BRI_WIDE_A=0: BM/8 boxes of 8 x 16, SWIZZLE_64B — twice the TMA ops)
//   B: one box of 16 (k) x BN (n) doubles, SWIZZLE_128B
// Fragment loads and bank conflicts: a 64-bit shared load is served one HALF-WARP at a time
// (16 lanes x 8 B = one 128-byte wavefront when the 16 addresses fall in 16 distinct 8-byte
// bank pairs; ncu: 2 wavefronts per LDS.64 at best).  With the textbook m16n8k4 mapping
// (fragment row g = lane / 4 <-> tile row g, fragment column g <-> tile column g) the 16 lanes
// of a half-warp (g = 0..3 or 4..7, t = lane % 4 = 0..3) read from only 64 of the 128 bytes of
// these swizzled rows, i.e. 4 wavefronts per load (profiles/r02_final_ncu_trsm_kernel_cfg3:
// every swizzled LDS.64 at 4.0 wavefronts, "ideal" 2.0).  FragMap<true> therefore permutes
// which tile row / column each fragment row / column stands for:
//     fragment row  g + 8h (h = 0, 1)  <->  tile row  (s & 1) + 8 (s >> 1) + 2 q + 4 h
//     fragment col  c                   <->  tile col  2 (c & 3) + (c >> 2)
// with g = 4 q + s.  A half-warp then covers all 16 bank pairs in both operand layouts
// (A: rows {0,1,8,9} + 2q + 4h under the XOR of k & 7 on 16-byte chunks; B: n & 7 = 2s + q
// XORed onto the chunk index k / 2).  Every output element still accumulates its k range in
// the same ascending k4 steps, so results are bit-identical to the textbook mapping; only the
// owner thread of each C element changes, which the epilogues account for through
// FragMap::row / FragMap::col.
#ifndef BRI_FRAG_PERM
#define BRI_FRAG_PERM 1
#endif
#pragma once

#include "bri_common.cuh"

#ifndef BRI_WIDE_A
#define BRI_WIDE_A 1
#endif

namespace bri {

constexpr int TILE_BK = 16;

template <int BM, int BN>
struct StageGeom {
  static constexpr int A_BYTES = BM * TILE_BK * 8;
  static constexpr int B_BYTES = BN * TILE_BK * 8;
  static constexpr int BYTES = A_BYTES + B_BYTES;
};

// Issue the TMA loads of one k-tile into stage buffer `st` (called by one lane).
// NBOX: the B operand arrives as NBOX boxes of BN / NBOX columns each through a narrower map (the
// [n][k] rows are 128 bytes, so consecutive boxes form the same swizzled layout as one wide box).
template <int BM, int BN, int NBOX = 1>
BRI_DEVI void tile_issue(uint8_t* st, uint64_t* full, const CUtensorMap* tmA, const CUtensorMap* tmB,
                         int a_row, int a_col, int a_slot, int b_row, int b_col, int b_slot) {
  mbar_arrive_expect_tx(full, StageGeom<BM, BN>::BYTES);
#if BRI_WIDE_A
#pragma unroll
  for (int ob = 0; ob < BM / 16; ++ob) tma_load_3d(st + ob * 2048, tmA, full, a_row + ob * 16, a_col, a_slot);
#else
#pragma unroll
  for (int ob = 0; ob < BM / 8; ++ob) tma_load_3d(st + ob * 1024, tmA, full, a_row + ob * 8, a_col, a_slot);
#endif
#pragma unroll
  for (int h = 0; h < NBOX; ++h)
    tma_load_3d(st + StageGeom<BM, BN>::A_BYTES + h * (StageGeom<BM, BN>::B_BYTES / NBOX), tmB, full, b_row,
                b_col + h * (BN / NBOX), b_slot);
}

// Tile row (0..15) of fragment row g + 8h and tile column (0..7) of fragment column c.
template <bool PERM>
struct FragMap {
  static BRI_DEVI int row(int g, int h) {
    return PERM ? ((g & 1) + ((g & 2) << 2) + ((g & 4) >> 1) + (h << 2)) : (g + (h << 3));
  }
  static BRI_DEVI int col(int c) { return PERM ? (((c & 3) << 1) + (c >> 2)) : c; }
};

// Warp-level accumulator of a (16*MI) x (8*NJ) sub-tile.  c[i][j][v] is the element at tile row
// 16 i + FragMap::row(lane / 4, v / 2), tile column 8 j + FragMap::col(2 (lane % 4) + (v & 1)).
template <int MI, int NJ, bool PERM = (BRI_FRAG_PERM != 0)>
struct WarpAcc {
  using Map = FragMap<PERM>;
  double c[MI][NJ][4];

  BRI_DEVI void zero() {
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int v = 0; v < 4; ++v) c[i][j][v] = 0.0;
  }

  // Consume one k-tile: A rows [wm0, wm0 + 16*MI), B cols [wn0, wn0 + 8*NJ).
  // Lanes whose k index is >= kvalid contribute zeros (K tail); FULL (a
  // whole k-tile is valid) drops those predicates.
  template <bool FULL = false>
  BRI_DEVI void mma_stage(const uint8_t* sA, const uint8_t* sB, int kvalid, int wm0, int wn0, int lane) {
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int kk = 0; kk < TILE_BK / 4; ++kk) {
      const int k = kk * 4 + t;
      const bool kin = FULL || k < kvalid;
      double a[MI][2], bf[NJ];
#if BRI_WIDE_A
      const uint32_t sw = (k & 7) << 4;
      const uint32_t off0 = k * 128 + ((Map::row(g, 0) * 8) ^ sw), off1 = k * 128 + ((Map::row(g, 1) * 8) ^ sw);
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const uint8_t* box = sA + ((wm0 + i * 16) >> 4) * 2048;
        a[i][0] = kin ? *reinterpret_cast<const double*>(box + off0) : 0.0;
        a[i][1] = kin ? *reinterpret_cast<const double*>(box + off1) : 0.0;
      }
#else
      static_assert(!PERM, "the permuted fragment map needs the 16-row A boxes");
      uint32_t offa = k * 64 + g * 8;
      offa ^= ((offa >> 7) & 3) << 4;
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int ob = (wm0 + i * 16) >> 3;
        a[i][0] = kin ? *reinterpret_cast<const double*>(sA + ob * 1024 + offa) : 0.0;
        a[i][1] = kin ? *reinterpret_cast<const double*>(sA + (ob + 1) * 1024 + offa) : 0.0;
      }
#endif
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int n = wn0 + j * 8 + Map::col(g);
        const uint32_t off = n * 128 + (((k >> 1) ^ (n & 7)) << 4) + ((k & 1) << 3);
        bf[j] = kin ? *reinterpret_cast<const double*>(sB + off) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma_16x8x4(c[i][j], a[i][0], a[i][1], bf[j]);
    }
  }

  // Scatter the accumulator into a column-major smem tile (element (r, c) at
  // tile[c * ldt + r]), optionally scaled.
  BRI_DEVI void to_smem(double* tile, int ldt, int wm0, int wn0, int lane, double alpha) const {
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int r = wm0 + i * 16 + Map::row(g, v >> 1);
          const int col = wn0 + j * 8 + Map::col(2 * t + (v & 1));
          tile[col * ldt + r] = alpha * c[i][j][v];
        }
  }
};

}  // namespace bri
