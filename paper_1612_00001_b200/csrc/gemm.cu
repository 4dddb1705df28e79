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

namespace bri {

namespace {

constexpr int BM = 128, BN = 128, BK = 16, STAGES = 4;
constexpr int NUM_CONSUMER_WARPS = 8;
constexpr int THREADS = NUM_CONSUMER_WARPS * 32;
constexpr int A_STAGE_BYTES = BM * BK * 8;  // 16 KB
constexpr int B_STAGE_BYTES = BN * BK * 8;  // 16 KB
constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

__global__ void __launch_bounds__(THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
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
      mbar_init(&empty[s], NUM_CONSUMER_WARPS);
    }
    fence_barrier_init();
  }
  __syncthreads();

  // Producer: lane 0 of warp 0 keeps the ring STAGES-1 k-tiles ahead.  Slot s
  // of k-tile kt is refilled for k-tile kt+STAGES once all 8 warps released it.
  const bool producer = (warp == 0 && lane == 0);
  auto issue = [&](int kt) {
    const int s = kt % STAGES;
    uint8_t* sA = smem + s * STAGE_BYTES;
    uint8_t* sB = sA + A_STAGE_BYTES;
    mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
    const int k0 = kt * BK;
#pragma unroll
    for (int ob = 0; ob < BM / 8; ++ob)
      tma_load_3d(sA + ob * 1024, &tmA, &full[s], p.a_r0 + m0 + ob * 8, p.a_c0 + k0, sa);
    tma_load_3d(sB, &tmB, &full[s], p.b_r0 + k0, p.b_c0 + n0, sb);
  };
  if (producer) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int kt = 0; kt < STAGES && kt < KT; ++kt) issue(kt);
  }

  // -------------------------------------------------------------- consumers
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp & 1;   // 2 warps along M (64 rows each)
  const int wn = warp >> 1;  // 4 warps along N (32 cols each)
  double acc[4][4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;

  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % STAGES;
    mbar_wait(&full[s], (kt / STAGES) & 1);
    const uint8_t* sA = smem + s * STAGE_BYTES;
    const uint8_t* sB = sA + A_STAGE_BYTES;
    const int kvalid = p.K - kt * BK;  // >= BK except on the tail tile
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      const int k = kk * 4 + t;
      const bool kin = k < kvalid;
      double a[4][2], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int ob = (wm * 64 + i * 16) >> 3;
        uint32_t off = k * 64 + g * 8;
        off ^= ((off >> 7) & 3) << 4;
        a[i][0] = kin ? *reinterpret_cast<const double*>(sA + ob * 1024 + off) : 0.0;
        a[i][1] = kin ? *reinterpret_cast<const double*>(sA + (ob + 1) * 1024 + off) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = wn * 32 + j * 8 + g;
        const uint32_t off = n * 128 + (((k >> 1) ^ (n & 7)) << 4) + ((k & 1) << 3);
        bf[j] = kin ? *reinterpret_cast<const double*>(sB + off) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_16x8x4(acc[i][j], a[i][0], a[i][1], bf[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    // refill the slot released one iteration ago (other warps are done with it by now)
    if (producer && kt >= 1) {
      const int kp = kt - 1;
      if (kp + STAGES < KT) {
        mbar_wait(&empty[kp % STAGES], (kp / STAGES) & 1);
        issue(kp + STAGES);
      }
    }
  }

  // -------------------------------------------------------------- epilogue
  double* cout = p.base + (long long)sc_out * p.slot_elems;
  const double* cin = p.base + (long long)sc_in * p.slot_elems;
  const bool read_c = p.beta != 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int row = m0 + wm * 64 + i * 16 + g + ((v >> 1) << 3);
        const int col = n0 + wn * 32 + j * 8 + 2 * t + (v & 1);
        if (row < p.M && col < p.N) {
          const long long off = (long long)(p.c_r0 + row) + (long long)(p.c_c0 + col) * p.ld;
          double r = p.alpha * acc[i][j][v];
          if (read_c) r = fma(p.beta, cin[off], r);
          cout[off] = r;
        }
      }
    }
  }
}

}  // namespace

int gemm_smem_bytes() { return SMEM_BYTES; }

cudaError_t launch_gemm(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmParams& p0,
                        int count, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (p0.M <= 0 || p0.N <= 0 || count <= 0) return cudaSuccess;
  GemmParams p = p0;
  p.tiles_m = (p.M + BM - 1) / BM;
  p.tiles_n = (p.N + BN - 1) / BN;
  if (p.K <= 0) {
    // C_out = beta * C_in: handled by the scale kernel (no products)
    return launch_scale_copy(p, count, stream);
  }
  dim3 grid(p.tiles_m * p.tiles_n, count);
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
  scale_copy_kernel<<<grid, 256, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace bri
