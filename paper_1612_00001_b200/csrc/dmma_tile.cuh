// Reusable pieces of the TMA -> smem -> DMMA tile pipeline shared by the GEMM
// (gemm.cu) and the fused triangular solve (trsm.cu).
//
// smem stage layout for a BM x BN output tile and BK = 16:
//   A: BM/16 boxes of 16 (m) x 16 (k) doubles, SWIZZLE_128B, 2 KB each
//      (BRI_WIDE_A=0: BM/8 boxes of 8 x 16, SWIZZLE_64B — twice the TMA ops)
//   B: one box of 16 (k) x BN (n) doubles, SWIZZLE_128B
// The swizzles make the m16n8k4 fragment loads conflict-free (2 wavefronts
// per 32 x 8 B request, the minimum).
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

// Warp-level accumulator of a (16*MI) x (8*NJ) sub-tile.
template <int MI, int NJ>
struct WarpAcc {
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
      const uint32_t off0 = k * 128 + ((g * 8) ^ sw), off1 = k * 128 + (((g + 8) * 8) ^ sw);
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const uint8_t* box = sA + ((wm0 + i * 16) >> 4) * 2048;
        a[i][0] = kin ? *reinterpret_cast<const double*>(box + off0) : 0.0;
        a[i][1] = kin ? *reinterpret_cast<const double*>(box + off1) : 0.0;
      }
#else
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
        const int n = wn0 + j * 8 + g;
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
          const int r = wm0 + i * 16 + g + ((v >> 1) << 3);
          const int col = wn0 + j * 8 + 2 * t + (v & 1);
          tile[col * ldt + r] = alpha * c[i][j][v];
        }
  }
};

}  // namespace bri
