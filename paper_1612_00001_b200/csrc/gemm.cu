// K1: batched FP64 GEMM with fused epilogue, sm_100a.
//
//   C_out = beta * C_in + alpha * A * B        (column-major "X-world", NN)
//
// Replaces the reference's `multiply` (dgemm through `x @ y`, core.py:173-181)
// and the in-place `subtract` that always follows it in `_fold`
// (engine.py:174-179): with alpha = -1, beta = 1 the Schur update
// r - l*t is one kernel and the product never round-trips through HBM.
// The same kernel does the trailing updates of the blocked LU and of the
// recursive triangular solves.
//
// Design (B200):
//  * FP64 tensor math on sm_100a is warp-level mma.sync only (tcgen05 has no
//    f64 kind); each m16n8k4 lowers to two SASS DMMA.8x8x4.
//  * Operands are staged by TMA (cp.async.bulk.tensor) into a 4-stage smem
//    ring guarded by full/empty mbarriers; one elected lane issues TMA
//    STAGES-1 k-tiles ahead while eight warps run DMMA (a dedicated producer
//    warp would cost 40+ registers per thread through allocation granularity).  Swizzles are chosen so every DMMA
//    fragment load is a 2-wavefront (conflict-free) LDS.64:
//      A tile (BM x BK, m contiguous) as 16 boxes of 8(m) x 16(k), SWIZZLE_64B
//      B tile (BK x BN, k contiguous) as 1 box of 16(k) x 128(n), SWIZZLE_128B
//  * All operands live in a slot arena (uniform b x b, ld) addressed through
//    one 3-D tensor map (rows, cols, slot); the batch index picks slots, so a
//    whole DAG level runs as one launch.  OOB boxes are zero-filled by TMA.
//  * Accumulation order per output element is fixed (k ascending in DMMA
//    k=4 chunks) and independent of batch size / grid, so results are
//    bit-reproducible across schedules.
#include "bri_common.cuh"
#include "bri_internal.h"
#include "dmma_tile.cuh"

#include <cstdlib>

namespace bri {

namespace {

#ifndef BRI_GEMM_PERM
// Fragment map of the 128 x 128 GEMM (dmma_tile.cuh): the permuted, bank-conflict-free map halves its
// LDS wavefronts, but the kernel is DMMA-bound (shared pipe 46% with the conflicts) and measured no
// faster with it (b = 1024 level batch 9.60 vs 9.56 ms, config 3 925 vs 923 ms), so it keeps the textbook
// map; the triangular-solve leaf, which is not, uses the permuted one.  Bits are identical either way.
#define BRI_GEMM_PERM 0
#endif
#ifndef BRI_GEMM_STAGES
#define BRI_GEMM_STAGES 4
#endif
constexpr int BM = 128, BN = 128, BK = TILE_BK, STAGES = BRI_GEMM_STAGES;
// 16 warps in a 4 x 4 grid, 32 x 32 warp tiles: four warps per scheduler hide
// DMMA / LDS latency (8 warps of 64 x 32 tiles left the DMMA pipe ~80% busy).
constexpr int WARPS_M = 4, WARPS_N = 4;
constexpr int NUM_WARPS = WARPS_M * WARPS_N;
constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
constexpr int THREADS = NUM_WARPS * 32;
constexpr int STAGE_BYTES = StageGeom<BM, BN>::BYTES;    // 32 KB
constexpr int LDT = BM + 4;                              // epilogue tile stride (doubles)
constexpr int TILE_BYTES = BN * LDT * 8;                 // 132 KB, reuses the stage ring
constexpr int RING_BYTES = STAGES * STAGE_BYTES > TILE_BYTES ? STAGES * STAGE_BYTES : TILE_BYTES;
constexpr int SMEM_BYTES = RING_BYTES + 1024 /*align*/ + 256 /*barriers*/;

// Tile geometry of the one-tile-per-CTA kernel: 128 x BNT tiles, 4 x WNT warps of 32 x 32.
//   <128, 4>: 512 threads, one CTA per SM (132 KB epilogue tile) — the long-K node GEMMs;
//   < 64, 2>: 256 threads, TWO CTAs per SM (96 KB ring each): while one CTA streams its C tile
//             (the epilogue is ~30% of a K = 128 tile and nothing hides it at one CTA per SM) the
//             other one's DMMA loop owns the tensor pipe — the LU's rank-128 trailing updates.
// Same per-element operation order in both (k ascending in k4 steps, then fma(beta, C_in, alpha * acc)).
template <int BNT, int WNT>
struct GemmGeom {
  static constexpr int BN = BNT, WARPS_N = WNT, NUM_WARPS = WARPS_M * WNT, THREADS = NUM_WARPS * 32;
  static constexpr int CTAS_PER_SM = BNT >= 128 ? 1 : 2;
  static constexpr int NBOX = BNT >= 128 ? 1 : BNT / 32;   // narrow tiles load B through the 32-column map
  static constexpr int STAGE_BYTES = StageGeom<BM, BNT>::BYTES;
  static constexpr int TILE_BYTES = BNT * LDT * 8;
  static constexpr int RING_BYTES = STAGES * STAGE_BYTES > TILE_BYTES ? STAGES * STAGE_BYTES : TILE_BYTES;
  static constexpr int SMEM_BYTES = RING_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

template <int BNT, int WNT>
__global__ void __launch_bounds__((GemmGeom<BNT, WNT>::THREADS), (GemmGeom<BNT, WNT>::CTAS_PER_SM))
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                GemmParams p) {
  using G = GemmGeom<BNT, WNT>;
  constexpr int BN = G::BN, NUM_WARPS = G::NUM_WARPS, STAGE_BYTES = G::STAGE_BYTES, RING_BYTES = G::RING_BYTES;
  constexpr int WTN = BN / G::WARPS_N;
  static_assert(WTN == 32 && WTM == 32, "32 x 32 warp tiles");
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned (TMA 128B swizzle atoms) by pointer arithmetic on the
  // __shared__ array, so the compiler keeps the shared address space (LDS, not
  // generic LD with 64-bit address math) for every fragment load
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + RING_BYTES);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int item = blockIdx.y;
  const int* it = p.items + 4 * item;
  const int sa = it[0], sb = it[1], sc_in = it[2], sc_out = it[3];
  const int tm = blockIdx.x % p.tiles_m;
  const int tn = blockIdx.x / p.tiles_m;
  const int m0 = tm * BM, n0 = tn * BN;
  const int KT = (p.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NUM_WARPS);
    }
    fence_barrier_init();
  }
  __syncthreads();

  // Producer: lane 0 of warp 0 keeps the ring STAGES-1 k-tiles ahead; the slot
  // of k-tile kt is refilled (for kt + STAGES) once all warps released it.
  const bool producer = (warp == 0 && lane == 0);
  auto issue = [&](int kt) {
    const int s = kt % STAGES;
    tile_issue<BM, BN, G::NBOX>(smem + s * STAGE_BYTES, &full[s], &tmA, &tmB, p.a_r0 + m0, p.a_c0 + kt * BK, sa,
                       p.b_r0 + kt * BK, p.b_c0 + n0, sb);
  };
  if (producer) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int kt = 0; kt < STAGES && kt < KT; ++kt) issue(kt);
  }

  const int wm0 = (warp % WARPS_M) * WTM;
  const int wn0 = (warp / WARPS_M) * WTN;
  WarpAcc<WTM / 16, WTN / 8, (BRI_GEMM_PERM != 0)> acc;
  acc.zero();
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % STAGES;
    mbar_wait(&full[s], (kt / STAGES) & 1);
    const uint8_t* sA = smem + s * STAGE_BYTES;
    if (p.K - kt * BK >= BK)
      acc.template mma_stage<true>(sA, sA + StageGeom<BM, BN>::A_BYTES, BK, wm0, wn0, lane);
    else
      acc.mma_stage(sA, sA + StageGeom<BM, BN>::A_BYTES, p.K - kt * BK, wm0, wn0, lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (producer && kt >= 1) {
      const int kp = kt - 1;
      if (kp + STAGES < KT) {
        mbar_wait(&empty[kp % STAGES], (kp / STAGES) & 1);
        issue(kp + STAGES);
      }
    }
  }

  // ------------------------------------------------------------ epilogue
  // Stage alpha*acc through smem, then stream whole columns (contiguous in
  // memory): every warp access is one 256 B run, and the C_in loads of two
  // columns are in flight together (C_in may alias C_out).
  __syncthreads();
  double* tile = reinterpret_cast<double*>(smem);
  acc.to_smem(tile, LDT, wm0, wn0, lane, p.alpha);
  __syncthreads();
  double* cout = p.base + (long long)sc_out * p.slot_elems;
  const double* cin = p.base + (long long)sc_in * p.slot_elems;
  const bool read_c = p.beta != 0.0;
  for (int c = warp; c < BN; c += 2 * NUM_WARPS) {
    double v[2][4], old[2][4];
    long long off[2][4];
    bool ok[2][4];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int col = c + u * NUM_WARPS;
      const int gcol = n0 + col;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int row = lane + 32 * q;
        const int grow = m0 + row;
        ok[u][q] = grow < p.M && gcol < p.N;
        off[u][q] = (long long)(p.c_r0 + grow) + (long long)(p.c_c0 + gcol) * p.ld;
        v[u][q] = tile[col * LDT + row];
        old[u][q] = (ok[u][q] && read_c) ? cin[off[u][q]] : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (ok[u][q]) cout[off[u][q]] = read_c ? fma(p.beta, old[u][q], v[u][q]) : v[u][q];
  }
}


// Persistent variant: tiles dealt round-robin over a capped grid (used when a
// concurrent critical path must keep SMs, e.g. the LU's bulk trailing update).
__global__ void __launch_bounds__(THREADS, 1)
    gemm_persistent_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned (TMA 128B swizzle atoms) by pointer arithmetic on the
  // __shared__ array, so the compiler keeps the shared address space (LDS, not
  // generic LD with 64-bit address math) for every fragment load
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + RING_BYTES);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int KT = (p.K + BK - 1) / BK;
  const int tiles_per_item = p.tiles_m * p.tiles_n;
  const int total = tiles_per_item * p.count;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NUM_WARPS);
    }
    fence_barrier_init();
  }
  __syncthreads();
  // Producer: lane 0 of warp 0 keeps the ring STAGES-1 k-tiles ahead; the slot
  // of k-tile kt is refilled (for kt + STAGES) once all warps released it.
  const bool producer = (warp == 0 && lane == 0);
  if (producer) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  const int wm0 = (warp % WARPS_M) * WTM;
  const int wn0 = (warp / WARPS_M) * WTN;

  // Tiles are dealt round-robin over the grid (one per CTA unless the launch
  // caps the CTA count, e.g. to leave SMs to a concurrent critical path); the
  // ring position g0 and its mbarrier phases run on across a CTA's tiles.
  int g0 = 0;
  auto issue_tile = [&](int tile, int kt, int gbase) {
    const int item = tile / tiles_per_item, rem = tile % tiles_per_item;
    const int* it = p.items + 4 * item;
    const int m0 = (rem % p.tiles_m) * BM, n0 = (rem / p.tiles_m) * BN;
    const int s = (gbase + kt) % STAGES;
    tile_issue<BM, BN>(smem + s * STAGE_BYTES, &full[s], &tmA, &tmB, p.a_r0 + m0, p.a_c0 + kt * BK, it[0],
                       p.b_r0 + kt * BK, p.b_c0 + n0, it[1]);
  };
  // the first STAGES k-tiles of a tile, each once its ring slot is released
  auto issue_head = [&](int tile, int gbase) {
    for (int kt = 0; kt < STAGES && kt < KT; ++kt) {
      const int gg = gbase + kt;
      if (gg >= STAGES) mbar_wait(&empty[gg % STAGES], ((gg / STAGES) - 1) & 1);
      issue_tile(tile, kt, gbase);
    }
  };
  if (producer && blockIdx.x < total) issue_head(blockIdx.x, 0);
  for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
    const int item = tile / tiles_per_item, rem = tile % tiles_per_item;
    const int* it = p.items + 4 * item;
    const int sc_in = it[2], sc_out = it[3];
    const int tm = rem % p.tiles_m;
    const int tn = rem / p.tiles_m;
    const int m0 = tm * BM, n0 = tn * BN;
    WarpAcc<WTM / 16, WTN / 8, (BRI_GEMM_PERM != 0)> acc;
    acc.zero();
    for (int kt = 0; kt < KT; ++kt) {
      const int gg = g0 + kt, s = gg % STAGES;
      mbar_wait(&full[s], (gg / STAGES) & 1);
      const uint8_t* sA = smem + s * STAGE_BYTES;
      if (p.K - kt * BK >= BK)
        acc.template mma_stage<true>(sA, sA + StageGeom<BM, BN>::A_BYTES, BK, wm0, wn0, lane);
      else
        acc.mma_stage(sA, sA + StageGeom<BM, BN>::A_BYTES, p.K - kt * BK, wm0, wn0, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (producer && kt >= 1) {
        const int kp = kt - 1;
        if (kp + STAGES < KT) {
          const int gp = g0 + kp;
          mbar_wait(&empty[gp % STAGES], (gp / STAGES) & 1);
          issue_tile(tile, kp + STAGES, g0);
        }
      }
    }
    g0 += KT;
    double* cout = p.base + (long long)sc_out * p.slot_elems;
    const double* cin = p.base + (long long)sc_in * p.slot_elems;
    const bool read_c = p.beta != 0.0;
    if (p.overlap) {
      // the next tile's first k-tiles load while this tile's epilogue runs
      if (producer && tile + (int)gridDim.x < total) issue_head(tile + gridDim.x, g0);
      // epilogue straight from the accumulators: per store instruction a warp writes
      // 4 columns x 8 contiguous rows (whole 32-byte sectors); same arithmetic as the
      // staged path, fma(beta, C_in, alpha * acc).  C_in may alias C_out: every element
      // is read and written by the same thread.
      const int g = lane >> 2, t = lane & 3;
      constexpr int JC = 2;   // fragment columns per round trip (register budget: 128 per thread)
#pragma unroll
      for (int i = 0; i < WTM / 16; ++i)
#pragma unroll
      for (int j0 = 0; j0 < WTN / 8; j0 += JC) {
        double old[JC][4];
#pragma unroll
        for (int j = 0; j < JC; ++j)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int grow = m0 + wm0 + 16 * i + decltype(acc)::Map::row(g, v >> 1);
            const int gcol = n0 + wn0 + 8 * (j0 + j) + decltype(acc)::Map::col(2 * t + (v & 1));
            const bool ok = grow < p.M && gcol < p.N;
            old[j][v] = (ok && read_c) ? cin[(long long)(p.c_r0 + grow) + (long long)(p.c_c0 + gcol) * p.ld] : 0.0;
          }
#pragma unroll
        for (int j = 0; j < JC; ++j)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int grow = m0 + wm0 + 16 * i + decltype(acc)::Map::row(g, v >> 1);
            const int gcol = n0 + wn0 + 8 * (j0 + j) + decltype(acc)::Map::col(2 * t + (v & 1));
            if (grow < p.M && gcol < p.N) {
              const double val = p.alpha * acc.c[i][j0 + j][v];
              cout[(long long)(p.c_r0 + grow) + (long long)(p.c_c0 + gcol) * p.ld] =
                  read_c ? fma(p.beta, old[j][v], val) : val;
            }
          }
      }
      continue;
    }

    // ---------------------------------------------------------- epilogue
    // Stage alpha*acc through smem, then stream whole columns (contiguous in
    // memory): every warp access is one 256 B run, and the C_in loads of two
    // columns are in flight together (C_in may alias C_out).
    __syncthreads();
    double* tile_s = reinterpret_cast<double*>(smem);
    acc.to_smem(tile_s, LDT, wm0, wn0, lane, p.alpha);
    __syncthreads();
    for (int c = warp; c < BN; c += 2 * NUM_WARPS) {
      double v[2][4], old[2][4];
      long long off[2][4];
      bool ok[2][4];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int col = c + u * NUM_WARPS;
        const int gcol = n0 + col;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int row = lane + 32 * q;
          const int grow = m0 + row;
          ok[u][q] = grow < p.M && gcol < p.N;
          off[u][q] = (long long)(p.c_r0 + grow) + (long long)(p.c_c0 + gcol) * p.ld;
          v[u][q] = tile_s[col * LDT + row];
          old[u][q] = (ok[u][q] && read_c) ? cin[off[u][q]] : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (ok[u][q]) cout[off[u][q]] = read_c ? fma(p.beta, old[u][q], v[u][q]) : v[u][q];
    }
    // the next tile's TMA writes (async proxy) reuse this smem
    fence_proxy_async_smem();
    __syncthreads();
    if (producer && tile + (int)gridDim.x < total) issue_head(tile + gridDim.x, g0);
  }
}

// ------------------------------------------------------------ skinny
// Short-K updates (K <= 128: the rank-32 / rank-128 updates inside the
// blocked LU) on 64 x 64 tiles: four times the CTAs of a 128 x 128 tile, no
// TMA pipeline to fill, operands staged in 32-wide k chunks with plain
// coalesced loads.  The DMMA sequence per output element (k ascending in
// m16n8k4 steps from a zero accumulator, then fma(beta, C_in, alpha * acc))
// is the big kernel's, so both paths give bit-identical results.
constexpr int SK_BM = 64, SK_BN = 64, SK_KC = 32;
constexpr int SK_LDA = SK_BM + 4;   // As[k][m]: 32 bytes mod 128 per k row, half-warp conflict-free (dmma_tile.cuh)
constexpr int SK_LDB = SK_KC + 4;   // Bs[n][k]: B fragments 2 wavefronts

__global__ void __launch_bounds__(256) skinny_kernel(GemmParams p) {
  __shared__ double As[SK_KC * SK_LDA];
  __shared__ double Bs[SK_BN * SK_LDB];
  if (p.early) pdl_trigger();
  pdl_wait();
  const int* it = p.items + 4 * blockIdx.y;
  const double* A = p.base + (long long)it[0] * p.slot_elems;
  const double* B = p.base + (long long)it[1] * p.slot_elems;
  const double* cin = p.base + (long long)it[2] * p.slot_elems;
  double* cout = p.base + (long long)it[3] * p.slot_elems;
  const int m0 = (blockIdx.x % p.tiles_m) * SK_BM, n0 = (blockIdx.x / p.tiles_m) * SK_BN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int wm0 = (warp & 1) * 32, wn0 = (warp >> 1) * 16;   // 2 x 4 warps, 32 x 16 each
  double acc[2][2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;
  for (int k0 = 0; k0 < p.K; k0 += SK_KC) {
    // A chunk: SK_KC columns of 64 contiguous rows; B chunk: 64 columns of SK_KC contiguous k
    for (int e = threadIdx.x; e < SK_KC * SK_BM; e += blockDim.x) {
      const int kk = e / SK_BM, m = e % SK_BM;
      const bool ok = m0 + m < p.M && k0 + kk < p.K;
      As[kk * SK_LDA + m] = ok ? A[(long long)(p.a_r0 + m0 + m) + (long long)(p.a_c0 + k0 + kk) * p.ld] : 0.0;
    }
    for (int e = threadIdx.x; e < SK_BN * SK_KC; e += blockDim.x) {
      const int n = e / SK_KC, kk = e % SK_KC;
      const bool ok = n0 + n < p.N && k0 + kk < p.K;
      Bs[n * SK_LDB + kk] = ok ? B[(long long)(p.b_r0 + k0 + kk) + (long long)(p.b_c0 + n0 + n) * p.ld] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SK_KC; kk += 4) {
      double a[2][2], b[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        a[i][0] = As[(kk + t) * SK_LDA + wm0 + 16 * i + g];
        a[i][1] = As[(kk + t) * SK_LDA + wm0 + 16 * i + g + 8];
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = Bs[(wn0 + 8 * j + g) * SK_LDB + kk + t];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_16x8x4(acc[i][j], a[i][0], a[i][1], b[j]);
    }
    __syncthreads();
  }
  // all C_in loads first (C_in may alias C_out): one round trip, not sixteen
  const bool read_c = p.beta != 0.0;
  double old[2][2][4];
  long long off[2][2][4];
  bool ok[2][2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int row = m0 + wm0 + 16 * i + g + ((v >> 1) << 3);
        const int col = n0 + wn0 + 8 * j + 2 * t + (v & 1);
        ok[i][j][v] = row < p.M && col < p.N;
        off[i][j][v] = (long long)(p.c_r0 + row) + (long long)(p.c_c0 + col) * p.ld;
        old[i][j][v] = (ok[i][j][v] && read_c) ? cin[off[i][j][v]] : 0.0;
      }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (ok[i][j][v]) {
          const double val = p.alpha * acc[i][j][v];
          cout[off[i][j][v]] = read_c ? fma(p.beta, old[i][j][v], val) : val;
        }
}

}  // namespace

int gemm_smem_bytes() { return SMEM_BYTES; }

// Dispatch thresholds for the short-K kernel (env overrides for tuning runs).
static int env_int(const char* name, int dflt) {
  const char* s = getenv(name);
  return (s && *s) ? atoi(s) : dflt;
}
int skinny_max_k() {
  static const int v = env_int("BRI_SKINNY_MAXK", 128);
  return v;
}
long long skinny_max_tiles() {
  static const long long v = env_int("BRI_SKINNY_MAXTILES", 148);   // 128x128 tiles (x batch) below one wave
  return v;
}

cudaError_t configure_gemm() {
  cudaError_t e = cudaFuncSetAttribute(gemm_kernel<128, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       GemmGeom<128, 4>::SMEM_BYTES);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(gemm_kernel<64, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             GemmGeom<64, 2>::SMEM_BYTES);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(gemm_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  return e;
}

cudaError_t launch_gemm(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmB32,
                        const GemmParams& p0, int count, cudaStream_t stream) {
  if (p0.M <= 0 || p0.N <= 0 || count <= 0) return cudaSuccess;
  GemmParams p = p0;
  p.tiles_m = (p.M + BM - 1) / BM;
  p.tiles_n = (p.N + BN - 1) / BN;
  if (p.K <= 0) {
    // C_out = beta * C_in: handled by the scale kernel (no products)
    return launch_scale_copy(p, count, stream);
  }
  if (p.K <= skinny_max_k() && (long long)p.tiles_m * p.tiles_n * count < skinny_max_tiles()) {
    GemmParams q = p;
    q.tiles_m = (p.M + SK_BM - 1) / SK_BM;
    q.tiles_n = (p.N + SK_BN - 1) / SK_BN;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(q.tiles_m * q.tiles_n, count);
    cfg.blockDim = dim3(256);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    pdl_attr(attr[0]);
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    count_launch();
    return cudaLaunchKernelEx(&cfg, skinny_kernel, q);
  }
  p.count = count;
  long long ctas = (long long)p.tiles_m * p.tiles_n * count;
  // opt-in (BRI_GEMM_OVERLAP=1): measured slower — level batch of 148 b=1024 nodes 9.77 vs
  // 9.56 ms, config 3 1031 vs 1016 ms: the register epilogue's 64-byte column pieces cost
  // more than the ~4% of a K=1024 tile the overlap could hide
  static const int overlap_env = env_int("BRI_GEMM_OVERLAP", 0);
  static const int num_sms = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  // overlapped persistent launch: more than one wave, nothing concurrent (caller's flag)
  p.overlap = (p.overlap && overlap_env && p.max_ctas <= 0 && ctas > num_sms) ? 1 : 0;
  if (p.overlap) {
    count_launch();
    gemm_persistent_kernel<<<dim3((unsigned)num_sms), THREADS, SMEM_BYTES, stream>>>(tmA, tmB, p);
    return cudaGetLastError();
  }
  if (p.max_ctas > 0 && ctas > p.max_ctas) ctas = p.max_ctas;
  if (ctas > 0x7fffffffLL) return cudaErrorInvalidValue;
  count_launch();
  // capped launches of short-K updates (the LU's rank-128 trailing and fold GEMMs next to the
  // pivot chain): a CTA's next tile starts loading during its epilogue (BRI_CAP_OVERLAP)
  static const int cap_overlap = env_int("BRI_CAP_OVERLAP", 0);
  if (ctas < (long long)p.tiles_m * p.tiles_n * count) {
    p.overlap = (cap_overlap && p.K <= cap_overlap) ? 1 : 0;
    gemm_persistent_kernel<<<dim3((unsigned)ctas), THREADS, SMEM_BYTES, stream>>>(tmA, tmB, p);
  } else {
    // 128 x 64 tiles, two CTAs per SM, for every K (BRI_GEMM_N64_MAXK=0 restores the 128 x 128
    // tiles; = k: only products with K <= k).  Measured on 444-item b = 1024 batches, TFLOP/s
    // 128x128 -> 128x64: K = 128 24.0 -> 28.4, K = 256 29.1 -> 32.4, K = 512 31.6 -> 33.5,
    // K = 1024 33.3 -> 34.1; config 3 923 -> 886 ms; bit-identical results.  A 3-stage ring and
    // the permuted fragment map were measured on it too: no gain (906.3 / 908.5 vs 906.5 ms at
    // BRI_GEMM_N64_MAXK=256).
    static const int n64_maxk = env_int("BRI_GEMM_N64_MAXK", 1 << 30);
    if (p.K <= n64_maxk) {
      using G = GemmGeom<64, 2>;
      p.tiles_n = (p.N + G::BN - 1) / G::BN;
      if ((long long)p.tiles_m * p.tiles_n > 0x7fffffffLL) return cudaErrorInvalidValue;
      gemm_kernel<64, 2><<<dim3(p.tiles_m * p.tiles_n, count), G::THREADS, G::SMEM_BYTES, stream>>>(tmA, tmB32, p);
    } else {
      gemm_kernel<128, 4><<<dim3(p.tiles_m * p.tiles_n, count), THREADS, SMEM_BYTES, stream>>>(tmA, tmB, p);
    }
  }
  return cudaGetLastError();
}

// C_out = beta * C_in over an M x N window (K == 0 degenerate product).
__global__ void scale_copy_kernel(GemmParams p) {
  const int* it = p.items + 4 * blockIdx.y;
  double* cout = p.base + (long long)it[3] * p.slot_elems;
  const double* cin = p.base + (long long)it[2] * p.slot_elems;
  const long long total = (long long)p.M * p.N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(e % p.M), col = (int)(e / p.M);
    const long long off = (long long)(p.c_r0 + row) + (long long)(p.c_c0 + col) * p.ld;
    cout[off] = p.beta == 0.0 ? 0.0 : p.beta * cin[off];
  }
}

cudaError_t launch_scale_copy(const GemmParams& p, int count, cudaStream_t stream) {
  dim3 grid(64, count);
  count_launch();
  scale_copy_kernel<<<grid, 256, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace bri
