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

namespace bri {

namespace {

constexpr int BM = 128, BN = 128, BK = TILE_BK, STAGES = 4;
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

__global__ void __launch_bounds__(THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
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
    tile_issue<BM, BN>(smem + s * STAGE_BYTES, &full[s], &tmA, &tmB, p.a_r0 + m0, p.a_c0 + kt * BK, sa,
                       p.b_r0 + kt * BK, p.b_c0 + n0, sb);
  };
  if (producer) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int kt = 0; kt < STAGES && kt < KT; ++kt) issue(kt);
  }

  const int wm0 = (warp % WARPS_M) * WTM;
  const int wn0 = (warp / WARPS_M) * WTN;
  WarpAcc<WTM / 16, WTN / 8> acc;
  acc.zero();
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % STAGES;
    mbar_wait(&full[s], (kt / STAGES) & 1);
    const uint8_t* sA = smem + s * STAGE_BYTES;
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

}  // namespace

int gemm_smem_bytes() { return SMEM_BYTES; }

cudaError_t configure_gemm() {
  return cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
}

cudaError_t launch_gemm(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmParams& p0,
                        int count, cudaStream_t stream) {
  if (p0.M <= 0 || p0.N <= 0 || count <= 0) return cudaSuccess;
  GemmParams p = p0;
  p.tiles_m = (p.M + BM - 1) / BM;
  p.tiles_n = (p.N + BN - 1) / BN;
  if (p.K <= 0) {
    // C_out = beta * C_in: handled by the scale kernel (no products)
    return launch_scale_copy(p, count, stream);
  }
  dim3 grid(p.tiles_m * p.tiles_n, count);
  count_launch();
  gemm_kernel<<<grid, THREADS, SMEM_BYTES, stream>>>(tmA, tmB, p);
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
