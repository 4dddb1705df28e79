// K2: fused triangular solves with many right-hand sides, sm_100a.
//
// Replaces the two dtrsm sweeps inside LAPACK dgetrs (core.py:259; getrs
// solves L then U) — the "p^-1 * l" half of every Schur node and the final
// block inversion.  Design:
//
//  * Diagonal 64 x 64 blocks of L (unit) and U (non-unit) are inverted once
//    per factorization (dinv_kernel), so every block step becomes DMMA work.
//  * trsm_kernel: one CTA owns a 32-column panel of the right-hand side and
//    sweeps the block rows of the triangle in order.  Block row i:
//        acc  = T[i, done] * X[done, panel]        (TMA-fed DMMA, K grows with i)
//        X_i  = Tinv_ii * (B_i - acc)               (second DMMA from smem)
//    The panel's own earlier X rows are re-read through TMA after a
//    fence.proxy.async, so CTAs never synchronize with each other: a whole
//    solve (or a batch of them) is one launch with nrhs/32 * batch CTAs.
//  * Used as the leaf (<= 512 rows) of the recursive solve in capi.cu, whose
//    upper levels are large GEMMs.
#include "bri_common.cuh"
#include "bri_internal.h"
#include "dmma_tile.cuh"

namespace bri {

namespace {

constexpr int T = TRSM_BLOCK;      // 64
// Variants (right-hand-side columns per CTA, ring depth):
//   <32, 3>: large batches, two CTAs per SM;
//   <16, 4>: a grid of <= one CTA per SM at 32 columns (a single factor's solve)
//            is split twice as fine, again two CTAs per SM to hide the per-block-row latency.
constexpr int THREADS = 256;
// Tile strides of the second product (textbook fragment map): a half-warp (4 values of
// lane / 4 x 4 of lane % 4) must touch 16 distinct 8-byte bank pairs per 64-bit load, i.e. the
// stride must be 32 bytes mod 128 in both operand patterns (T + 8 left the Tinv loads at 4
// wavefronts per LDS.64 instead of 2).
constexpr int LDD = T + 4;         // Tinv tile stride ([k][m], A-operand pattern)
constexpr int LDR = T + 4;         // R tile stride ([n][k], B-operand pattern)
constexpr int LDB = T + 4;         // prefetched B_i tile stride ([n][k])
// DENSE: three CTAs per SM (<= 76,800 bytes each): the Tinv tile unpadded with an XOR swizzle on
// 32-byte groups (same half-warp property as the padded stride), the prefetched B_i tile shares the R
// buffer (R = B_i - acc is computed in place by the thread that owns each element) and the ring has
// two stages.
template <int BN, int STAGES, bool DENSE = false>
constexpr int smem_bytes() {
  return STAGES * StageGeom<T, BN>::BYTES + T * (DENSE ? T : LDD) * 8 + (DENSE ? 1 : 2) * BN * LDR * 8 + 1024 + 256;
}
template <bool DENSE>
BRI_DEVI int tinv_index(int k, int m) {
  return DENSE ? k * T + (m ^ ((k & 3) << 2)) : k * LDD + m;
}

BRI_DEVI void cp_async16(void* smem_dst, const void* gsrc, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem_dst)), "l"(gsrc),
               "r"(valid ? 16 : 0)
               : "memory");
}

// --------------------------------------------------------------- dinv
// Invert the T x T diagonal blocks of the factor in slot F: unit lower (L) or
// non-unit upper (U).  Outside [0, n) the block is the identity.  One CTA per
// block: the block is read once into smem, each of the 8 warps owns 8 columns of
// the inverse (lane l holds rows l and l + 32 of each) and runs their 8
// independent substitution chains interleaved (shuffles, no block barriers on
// the dependency chain).  Each column sees the same operation sequence as a
// one-column-per-warp sweep.  dinv layout per item: [nblk][T x T column-major].
__device__ __noinline__ double slow_div(double w, double t) { return w / t; }

constexpr int DINV_WARPS = 8;
constexpr int DINV_COLS = T / DINV_WARPS;   // columns per warp

// UNIT: the triangle's diagonal is taken as 1 (LU's L, or the Lᵀ of a transposed factor);
// otherwise its stored diagonal is used (U, or the Uᵀ of a transposed factor).
template <bool LOWER, bool UNIT = LOWER>
__global__ void __launch_bounds__(DINV_WARPS * 32) dinv_kernel(ArenaView a, const int* fslots, double* dinv,
                                                               int nblk, int blk0) {
  __shared__ double S[T][T + 1];   // S[c][r] = block(r, c)
  __shared__ double rd[T];         // non-unit: reciprocals of the diagonal
  const int blk = blk0 + blockIdx.x, item = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* F = a.base + (long long)fslots[item] * a.slot_elems;
  const int base = blk * T;
  for (int e = threadIdx.x; e < T * T; e += DINV_WARPS * 32) {
    const int r = e % T, cc = e / T;
    const int gi = base + r, gj = base + cc;
    double v = (gi < a.n && gj < a.n) ? F[gi + (long long)gj * a.ld] : (r == cc ? 1.0 : 0.0);
    if (UNIT && r == cc) v = 1.0;
    if (LOWER && r < cc) v = 0.0;
    if (!LOWER && r > cc) v = 0.0;
    S[cc][r] = v;
  }
  __syncthreads();
  // x_k = w_k / t_kk with the reciprocals computed once, all in parallel: q = w * r, then one
  // residual correction q + r * fma(-t, q, w) — with r = RN(1 / t) that is the correctly rounded
  // quotient (Markstein), i.e. the same bits as the IEEE division it replaces, but three dependent
  // operations on every column's chain instead of a ~100-cycle division subroutine per step (the
  // non-unit kernel took 7x the unit one; config 2: 138 us per U table on the critical path).
  // The plain product w * r rounds differently and moved BASELINE config 4's near-threshold
  // singular pivot from the reference's branch A/D/A/D to A/D/A.  Non-finite results (zero or
  // non-finite diagonal) take the division itself.
  if (!UNIT) {
    if (threadIdx.x < T) rd[threadIdx.x] = 1.0 / S[threadIdx.x][threadIdx.x];
    __syncthreads();
  }
  auto div_by = [](double w, double t, double r) {
    const double q = w * r;
    double q1 = fma(fma(-t, q, w), r, q);
    // NaN / Inf: the true division, out of line so that it is never speculated onto the chain
    if (!(fabs(q1) <= 1.79769313486231570e308)) q1 = slow_div(w, t);
    return q1;
  };
  double x0[DINV_COLS], x1[DINV_COLS];   // column c = warp + DINV_WARPS * q: rows lane, lane + 32
#pragma unroll
  for (int q = 0; q < DINV_COLS; ++q) {
    const int c = warp + DINV_WARPS * q;
    x0[q] = (lane == c) ? 1.0 : 0.0;
    x1[q] = (lane + 32 == c) ? 1.0 : 0.0;
  }
  if (LOWER) {
#pragma unroll 2
    for (int k = 0; k < T; ++k) {
      const double s0 = S[k][lane], s1 = S[k][lane + 32];
#pragma unroll
      for (int q = 0; q < DINV_COLS; ++q) {
        if (!UNIT) {   // x_k *= 1 / l_kk before it propagates (forward substitution, non-unit)
          const double rk = rd[k], dk = S[k][k];
          if (k >= 32) { if (lane == k - 32) x1[q] = div_by(x1[q], dk, rk); } else { if (lane == k) x0[q] = div_by(x0[q], dk, rk); }
        }
        if (UNIT && k == T - 1) continue;
        const double xk = __shfl_sync(0xffffffffu, k < 32 ? x0[q] : x1[q], k & 31);
        if (lane > k) x0[q] = fma(-s0, xk, x0[q]);
        if (lane + 32 > k) x1[q] = fma(-s1, xk, x1[q]);
      }
    }
  } else if (UNIT) {   // unit upper (Lᵀ): backward substitution without divisions
#pragma unroll 2
    for (int k = T - 1; k >= 0; --k) {
      const double s0 = S[k][lane], s1 = S[k][lane + 32];
#pragma unroll
      for (int q = 0; q < DINV_COLS; ++q) {
        const double xk = __shfl_sync(0xffffffffu, k < 32 ? x0[q] : x1[q], k & 31);
        if (lane < k) x0[q] = fma(-s0, xk, x0[q]);
        if (lane + 32 < k) x1[q] = fma(-s1, xk, x1[q]);
      }
    }
  } else {
#pragma unroll 2
    for (int k = T - 1; k >= 0; --k) {
      const double rk = rd[k], dk = S[k][k], s0 = S[k][lane], s1 = S[k][lane + 32];
#pragma unroll
      for (int q = 0; q < DINV_COLS; ++q) {
        if (k >= 32) { if (lane == k - 32) x1[q] = div_by(x1[q], dk, rk); } else { if (lane == k) x0[q] = div_by(x0[q], dk, rk); }
        const double xk = __shfl_sync(0xffffffffu, k < 32 ? x0[q] : x1[q], k & 31);
        if (lane < k) x0[q] = fma(-s0, xk, x0[q]);
        if (lane + 32 < k) x1[q] = fma(-s1, xk, x1[q]);
      }
    }
  }
  double* out = dinv + ((long long)item * nblk + blk) * T * T;
#pragma unroll
  for (int q = 0; q < DINV_COLS; ++q) {
    const int c = warp + DINV_WARPS * q;
    out[(long long)c * T + lane] = x0[q];
    out[(long long)c * T + lane + 32] = x1[q];
  }
}

// --------------------------------------------------------------- solve
struct TrsmArgs {
  double* base;
  int ld;
  long long slot_elems;
  const int* items;     // (F, W) per item
  const double* dinv;   // per item [nblk][T*T] (or per factor, through didx)
  const int* didx;      // optional: item -> index of its dinv table (solves sharing a factor)
  int nblk;
  int r0, nr, c_off, nrhs;
  int tri_rhs;          // LOWER only: right-hand side is unit-lower-triangular (an identity
                        // being inverted): rows above a column's diagonal are zero and stay zero
};

template <bool LOWER, int BN, int STAGES, bool DENSE = false>
__global__ void __launch_bounds__(THREADS, (DENSE ? 3 : 2))
    trsm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TrsmArgs p) {
  constexpr int SB = StageGeom<T, BN>::BYTES;
  constexpr int XJ = BN / 16;       // n8 tiles per warp (4 warps along M x 2 along N, 16 x BN/2 each)
  constexpr int NBOX = BN > 32 ? BN / 32 : 1;   // BN = 64 loads its X tiles as two 32-column boxes (tmB32)
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned (TMA 128B swizzle atoms) by pointer arithmetic on the
  // __shared__ array, so the compiler keeps the shared address space (LDS, not
  // generic LD with 64-bit address math) for every fragment load
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  double* D = reinterpret_cast<double*>(smem + STAGES * SB);   // Tinv_ii, [k][m] col-major (LDD)
  double* R = D + T * (DENSE ? T : LDD);                                // B_i - acc, [n][k] (LDR)
  double* Bst = DENSE ? R : R + BN * LDR;                               // prefetched B_i, [n][k] (LDB)
  uint64_t* full = reinterpret_cast<uint64_t*>(Bst + BN * LDB);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int item = blockIdx.y;
  const int fs = p.items[2 * item], ws = p.items[2 * item + 1];
  const int c0 = p.c_off + blockIdx.x * BN;
  const int cend = p.c_off + p.nrhs;
  double* W = p.base + (long long)ws * p.slot_elems;
  const double* dinv = p.dinv + (long long)(p.didx ? p.didx[item] : item) * p.nblk * T * T;
  const int nb = (p.nr + T - 1) / T;
  // both products: 4 warps along M x 2 along N, 16 x BN/2 each; every output
  // element accumulates its k range in ascending k4-steps (splitting k across
  // warps was measured no faster and changes the rounding near singular pivots)
  const int xm0 = (warp & 3) * 16, xn0 = (warp >> 2) * (BN / 2);
  const bool producer = (warp == 0 && lane == 0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], THREADS / 32);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (producer) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }

  int it = 0;   // k-tiles consumed so far (ring position / phase)
  int pre = 0;  // k-tiles of the current block row already issued during the previous one
  // first block row with nonzeros in this CTA's columns (triangular right-hand side)
  const int i0 = (LOWER && p.tri_rhs) ? max(0, (c0 - p.r0) / T) : 0;
  for (int ii = LOWER ? i0 : 0; ii < nb; ++ii) {
    const int i = LOWER ? ii : nb - 1 - ii;
    const int row0 = p.r0 + i * T;
    const int rows = min(T, p.r0 + p.nr - row0);
    const int klo = LOWER ? p.r0 + i0 * T : row0 + T;
    const int khi = LOWER ? row0 : p.r0 + p.nr;
    const int K = khi - klo;
    const int KT = K > 0 ? (K + TILE_BK - 1) / TILE_BK : 0;
    auto issue = [&](int kt) {
      const int s = (it + kt) % STAGES;
      tile_issue<T, BN, NBOX>(smem + s * SB, &full[s], &tmA, &tmB, row0, klo + kt * TILE_BK, fs,
                              klo + kt * TILE_BK, c0, ws);
    };
    if (producer)
      for (int kt = pre; kt < STAGES && kt < KT; ++kt) issue(kt);
    pre = 0;
    // prefetch Tinv_ii and B_i with cp.async; they land while the K loop runs
    {
      const double* Di = dinv + (long long)(row0 / T) * T * T;
      for (int e = threadIdx.x; e < T * T / 2; e += THREADS) {
        const int k = e / (T / 2), r2 = (e % (T / 2)) * 2;
        cp_async16(&D[tinv_index<DENSE>(k, r2)], Di + k * T + r2, true);
      }
      for (int e = threadIdx.x; e < BN * T / 2; e += THREADS) {
        const int cc = e / (T / 2), r2 = (e % (T / 2)) * 2;
        const bool ok = r2 < rows && c0 + cc < cend;
        const double* src = ok ? W + (long long)(row0 + r2) + (long long)(c0 + cc) * p.ld : W;
        cp_async16(&Bst[cc * LDB + r2], src, ok);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    WarpAcc<1, XJ> acc;
    acc.zero();
    for (int kt = 0; kt < KT; ++kt) {
      const int s = (it + kt) % STAGES;
      mbar_wait(&full[s], ((it + kt) / STAGES) & 1);
      const uint8_t* sA = smem + s * SB;
      if (K - kt * TILE_BK >= TILE_BK)
        acc.template mma_stage<true>(sA, sA + StageGeom<T, BN>::A_BYTES, TILE_BK, xm0, xn0, lane);
      else
        acc.mma_stage(sA, sA + StageGeom<T, BN>::A_BYTES, K - kt * TILE_BK, xm0, xn0, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (producer && kt >= 1) {
        const int kp = kt - 1;
        if (kp + STAGES < KT) {
          mbar_wait(&empty[(it + kp) % STAGES], ((it + kp) / STAGES) & 1);
          issue(kp + STAGES);
        }
      }
    }
    // (the epilogue's __syncthreads below ends every read of the ring before reuse)
    it += KT;
    // Lower sweep: the next block row's first k-tiles read only X rows finished
    // before this one, so they load while this row's epilogue runs (each ring
    // slot once its last reader released it).
    if (LOWER && producer && ii + 1 < nb) {
      const int row0n = row0 + T;
      const int KTn = (row0n - klo + TILE_BK - 1) / TILE_BK;
      const int safe = min(min(STAGES, KT), KTn);
      for (int kt = 0; kt < safe; ++kt) {
        const int q = it + kt;
        if (q >= STAGES) mbar_wait(&empty[q % STAGES], ((q / STAGES) - 1) & 1);
        tile_issue<T, BN, NBOX>(smem + (q % STAGES) * SB, &full[q % STAGES], &tmA, &tmB, row0n,
                                klo + kt * TILE_BK, fs, klo + kt * TILE_BK, c0, ws);
      }
      pre = safe;
    }

    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    // R = B_i - acc  (rows >= rows and columns >= nrhs are zero)
#pragma unroll
    for (int j = 0; j < XJ; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        // the accumulator's own (permuted) fragment map: see dmma_tile.cuh
        const int r = xm0 + decltype(acc)::Map::row(g, v >> 1);
        const int cc = xn0 + j * 8 + decltype(acc)::Map::col(2 * t + (v & 1));
        const bool ok = r < rows && c0 + cc < cend;
        R[cc * LDR + r] = ok ? Bst[cc * LDB + r] - acc.c[0][j][v] : 0.0;
      }
    __syncthreads();
    // X_i = Tinv_ii * R   (64 x BN x 64 DMMA from smem)
    double x[XJ][4];
#pragma unroll
    for (int j = 0; j < XJ; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) x[j][v] = 0.0;
#pragma unroll 4
    for (int k0 = 0; k0 < T; k0 += 4) {
      const double a0 = D[tinv_index<DENSE>(k0 + t, xm0 + g)];
      const double a1 = D[tinv_index<DENSE>(k0 + t, xm0 + g + 8)];
#pragma unroll
      for (int j = 0; j < XJ; ++j) {
        const double b0 = R[(xn0 + j * 8 + g) * LDR + k0 + t];
        dmma_16x8x4(x[j], a0, a1, b0);
      }
    }
#pragma unroll
    for (int j = 0; j < XJ; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int r = xm0 + g + ((v >> 1) << 3);
        const int cc = xn0 + j * 8 + 2 * t + (v & 1);
        if (r < rows && c0 + cc < cend) W[(long long)(row0 + r) + (long long)(c0 + cc) * p.ld] = x[j][v];
      }
    // the next block rows read these X rows through TMA (async proxy)
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
  }
}


// --------------------------------------------------------------- right solve
// X * U[J, J] = B in place on columns [J0, J0 + W) of slot G (all n rows),
// U from the factor in slot F with its inverted 64 x 64 diagonal blocks in
// `dinv` (dinv_kernel<false>): per 64-column block b,
//     X_b = (B_b - sum_{a < b} X_a U_ab) * Uinv_bb.
// Rows are independent, so one CTA owns RT_R rows and the whole block: the
// in-place update needs no cross-CTA ordering.  Used by the folded Schur
// update (capi.cu getrf_device): C = rt * U^-1, 128 columns per outer block.
constexpr int RT_R = 32;               // rows per CTA
constexpr int RT_THREADS = 128;        // 4 warps: 2 along M (16 rows) x 2 along N (32 cols)
constexpr int RT_LDX = RT_R + 4;       // [col][row] tiles (A-operand pattern: 32 bytes mod 128 per k row)
constexpr int RT_LDU = T + 4;          // [n][k] tiles (B-operand pattern)
constexpr int RT_SMEM = (3 * T * RT_LDX + T * RT_LDU) * 8;

struct RtrsmArgs {
  double* base;
  int ld, n;
  long long slot_elems;
  const int* items;      // (G, F) per item
  const double* dinv;    // per item [nblk][T*T], upper
  int nblk, J0, W;
};

__global__ void __launch_bounds__(RT_THREADS) rtrsm_kernel(RtrsmArgs p) {
  extern __shared__ double rt_smem[];
  double* Xs = rt_smem;                       // X_0, X_1: [col][row]
  double* As = Xs + 2 * T * RT_LDX;           // B_b - ..., [col][row]
  double* Us = As + T * RT_LDX;               // U_ab or Uinv_bb, [n][k]
  const int item = blockIdx.y, m0 = blockIdx.x * RT_R;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int wm0 = (warp & 1) * 16, wn0 = (warp >> 1) * 32;
  double* G = p.base + (long long)p.items[2 * item] * p.slot_elems;
  const double* F = p.base + (long long)p.items[2 * item + 1] * p.slot_elems;
  const double* dinv = p.dinv + (long long)item * p.nblk * T * T;
  const int nbw = (p.W + T - 1) / T;
  for (int b = 0; b < nbw; ++b) {
    const int cb = p.J0 + b * T, wb = min(T, p.W - b * T);
    for (int e = tid; e < T * RT_R; e += RT_THREADS) {
      const int r = e % RT_R, cc = e / RT_R;
      As[cc * RT_LDX + r] = (m0 + r < p.n && cc < wb) ? G[(m0 + r) + (long long)(cb + cc) * p.ld] : 0.0;
    }
    __syncthreads();
    double acc[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v)
        acc[j][v] = As[(wn0 + j * 8 + 2 * t + (v & 1)) * RT_LDX + wm0 + g + ((v >> 1) << 3)];
    for (int a = 0; a < b; ++a) {
      const int ra = p.J0 + a * T;
      for (int e = tid; e < T * T; e += RT_THREADS) {
        const int k = e % T, nn = e / T;
        Us[nn * RT_LDU + k] = nn < wb ? F[(ra + k) + (long long)(cb + nn) * p.ld] : 0.0;
      }
      __syncthreads();
      const double* Xa = Xs + a * T * RT_LDX;
#pragma unroll 4
      for (int k0 = 0; k0 < T; k0 += 4) {
        const double a0 = -Xa[(k0 + t) * RT_LDX + wm0 + g], a1 = -Xa[(k0 + t) * RT_LDX + wm0 + g + 8];
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_16x8x4(acc[j], a0, a1, Us[(wn0 + j * 8 + g) * RT_LDU + k0 + t]);
      }
      __syncthreads();
    }
    const double* Di = dinv + (long long)(cb / T) * T * T;
    for (int e = tid; e < T * T; e += RT_THREADS) {
      const int k = e % T, nn = e / T;
      Us[nn * RT_LDU + k] = Di[nn * T + k];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v)
        As[(wn0 + j * 8 + 2 * t + (v & 1)) * RT_LDX + wm0 + g + ((v >> 1) << 3)] = acc[j][v];
    __syncthreads();
    double x[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) x[j][v] = 0.0;
#pragma unroll 4
    for (int k0 = 0; k0 < T; k0 += 4) {
      const double a0 = As[(k0 + t) * RT_LDX + wm0 + g], a1 = As[(k0 + t) * RT_LDX + wm0 + g + 8];
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_16x8x4(x[j], a0, a1, Us[(wn0 + j * 8 + g) * RT_LDU + k0 + t]);
    }
    double* Xb = Xs + b * T * RT_LDX;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v)
        Xb[(wn0 + j * 8 + 2 * t + (v & 1)) * RT_LDX + wm0 + g + ((v >> 1) << 3)] = x[j][v];
    __syncthreads();
    for (int e = tid; e < T * RT_R; e += RT_THREADS) {
      const int r = e % RT_R, cc = e / RT_R;
      if (m0 + r < p.n && cc < wb) G[(m0 + r) + (long long)(cb + cc) * p.ld] = Xb[cc * RT_LDX + r];
    }
    // the next block's loads overwrite As / Us only after the barrier at its top
  }
}
}  // namespace

int trsm_smem_bytes() { return smem_bytes<32, 3>(); }

cudaError_t configure_trsm() {
  cudaError_t e = cudaSuccess;
  auto set = [&](const void* f, int bytes) {
    if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  };
  set((const void*)trsm_kernel<true, 32, 3>, smem_bytes<32, 3>());
  set((const void*)trsm_kernel<false, 32, 3>, smem_bytes<32, 3>());
  set((const void*)trsm_kernel<true, 64, 4>, smem_bytes<64, 4>());
  set((const void*)trsm_kernel<false, 64, 4>, smem_bytes<64, 4>());
  set((const void*)trsm_kernel<true, 16, 4>, smem_bytes<16, 4>());
  set((const void*)trsm_kernel<false, 16, 4>, smem_bytes<16, 4>());
  set((const void*)trsm_kernel<true, 32, 2, true>, smem_bytes<32, 2, true>());
  set((const void*)trsm_kernel<false, 32, 2, true>, smem_bytes<32, 2, true>());
  set((const void*)rtrsm_kernel, RT_SMEM);
  return e;
}

cudaError_t launch_rtrsm(const ArenaView& a, const int* gf, int count, const double* dinv_u, int J0, int W,
                         cudaStream_t s) {
  RtrsmArgs p;
  p.base = a.base;
  p.ld = a.ld;
  p.n = a.n;
  p.slot_elems = a.slot_elems;
  p.items = gf;
  p.dinv = dinv_u;
  p.nblk = (a.n + T - 1) / T;
  p.J0 = J0;
  p.W = W;
  count_launch();
  rtrsm_kernel<<<dim3((a.n + RT_R - 1) / RT_R, count), RT_THREADS, RT_SMEM, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_dinv_t(const ArenaView& a, const int* fslots, int count, bool lower, bool unit, double* dinv,
                          int blk0, int nblocks, cudaStream_t s) {
  if (lower == unit) return launch_dinv(a, fslots, count, lower, dinv, blk0, nblocks, s);
  const int nblk = (a.n + T - 1) / T;
  if (nblocks <= 0) nblocks = nblk - blk0;
  dim3 grid(nblocks, count);
  count_launch();
  if (lower)
    dinv_kernel<true, false><<<grid, DINV_WARPS * 32, 0, s>>>(a, fslots, dinv, nblk, blk0);
  else
    dinv_kernel<false, true><<<grid, DINV_WARPS * 32, 0, s>>>(a, fslots, dinv, nblk, blk0);
  return cudaGetLastError();
}

cudaError_t launch_dinv(const ArenaView& a, const int* fslots, int count, bool lower, double* dinv,
                        int blk0, int nblocks, cudaStream_t s) {
  const int nblk = (a.n + T - 1) / T;
  if (nblocks <= 0) nblocks = nblk - blk0;
  dim3 grid(nblocks, count);
  count_launch();
  if (lower)
    dinv_kernel<true><<<grid, DINV_WARPS * 32, 0, s>>>(a, fslots, dinv, nblk, blk0);
  else
    dinv_kernel<false><<<grid, DINV_WARPS * 32, 0, s>>>(a, fslots, dinv, nblk, blk0);
  return cudaGetLastError();
}

cudaError_t launch_trsm_fused(const CUtensorMap& tmA, const CUtensorMap& tmB32, const CUtensorMap& tmB16,
                              const ArenaView& a, const int* fw, int count, const double* dinv, bool lower, int r0,
                              int nr, int c_off, int nrhs, bool tri_rhs, cudaStream_t s, const int* didx) {
  TrsmArgs p;
  p.base = a.base;
  p.ld = a.ld;
  p.slot_elems = a.slot_elems;
  p.items = fw;
  p.dinv = dinv;
  p.didx = didx;
  p.nblk = (a.n + T - 1) / T;
  p.r0 = r0;
  p.nr = nr;
  p.c_off = c_off;
  p.nrhs = nrhs;
  p.tri_rhs = tri_rhs ? 1 : 0;
  static const int sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  bool fine = (long long)((nrhs + 31) / 32) * count <= sms;
  // BRI_TRSM_BN64: 1 = large batches (at least two CTAs of 64 columns per SM), 2 = always (tests)
  static const int wide_env = [] {
    const char* e = getenv("BRI_TRSM_BN64");
    return e != nullptr ? atoi(e) : 0;
  }();
  // BRI_TRSM_DENSE=1: large batches on the three-CTA-per-SM variant
  static const int dense_env = [] {
    const char* e = getenv("BRI_TRSM_DENSE");
    return e != nullptr ? atoi(e) : 0;
  }();
  // nr x nr triangle against nrhs columns (tri_rhs: column c starts at its diagonal)
  double per = (double)nr * nr * nrhs;
  if (tri_rhs) {
    double t = 0.0;
    for (int c = 0; c < nrhs; ++c) {
      const int top = (c_off + c) > r0 ? (c_off + c) - r0 : 0;
      const double h = top < nr ? (double)(nr - top) : 0.0;
      t += h * h;
    }
    per = t;
  }
  count_flops(FLOP_TRSM, per * count);
  count_launch();
  if (wide_env >= 2 && nrhs >= 64) fine = false;
  if (fine) {
    dim3 grid((nrhs + 15) / 16, count);
    if (lower) trsm_kernel<true, 16, 4><<<grid, THREADS, smem_bytes<16, 4>(), s>>>(tmA, tmB16, p);
    else trsm_kernel<false, 16, 4><<<grid, THREADS, smem_bytes<16, 4>(), s>>>(tmA, tmB16, p);
  } else if (wide_env && nrhs >= 64 && (wide_env >= 2 || (long long)((nrhs + 63) / 64) * count >= 2 * sms)) {
    // large batches: 64 columns per CTA (one CTA per SM) — half the T-tile traffic per flop and
    // 16 x 32 warp tiles (1.5 instead of 2 fragment loads per DMMA: ncu shows the 32-column
    // kernel at 73% of the shared-memory pipe with the DMMA pipe at 58-69%)
    dim3 grid((nrhs + 63) / 64, count);
    if (lower) trsm_kernel<true, 64, 4><<<grid, THREADS, smem_bytes<64, 4>(), s>>>(tmA, tmB32, p);
    else trsm_kernel<false, 64, 4><<<grid, THREADS, smem_bytes<64, 4>(), s>>>(tmA, tmB32, p);
  } else if (dense_env) {
    dim3 grid((nrhs + 31) / 32, count);
    if (lower) trsm_kernel<true, 32, 2, true><<<grid, THREADS, smem_bytes<32, 2, true>(), s>>>(tmA, tmB32, p);
    else trsm_kernel<false, 32, 2, true><<<grid, THREADS, smem_bytes<32, 2, true>(), s>>>(tmA, tmB32, p);
  } else {
    dim3 grid((nrhs + 31) / 32, count);
    if (lower) trsm_kernel<true, 32, 3><<<grid, THREADS, smem_bytes<32, 3>(), s>>>(tmA, tmB32, p);
    else trsm_kernel<false, 32, 3><<<grid, THREADS, smem_bytes<32, 3>(), s>>>(tmA, tmB32, p);
  }
  return cudaGetLastError();
}

}  // namespace bri
