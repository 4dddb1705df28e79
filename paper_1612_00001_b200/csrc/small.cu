// K6: fused one-CTA Schur node / block inverse for small blocks (n <= 96), sm_100a.
//
// For b <= 96 a whole node of the reference's `_fold` (engine.py:157-180) is
// one CTA's work: the pivot solve W = P^-1 * l with partial pivoting (dgetrf
// pivot decisions on the X-world view, core.py:249, and the growth-scaled
// singularity test of core.py:200-209) and the fused update out = r - rt * W
// on the tensor cores, in one launch per DAG level, one CTA per node.  This is
// the latency-bound regime of BASELINE config 1 (b = 64) and of every small-b
// case in the reference's own test suite.
//
// In X-world the node computes  out^ = r^ - rt^ * (p^)^-1 * l^  which is the
// transpose of the reference's  r - l @ (inv(p) @ rt)  (all hats are the
// column-major views of the row-major blocks).
//
// Design (latency first — a 64 x 64 node is ~0.8 MFLOP, nothing to stream):
//  * The augmented matrix [p^ | l^] (N x 2N) lives in REGISTERS: lane owns rows
//    lane + 32h, warp w owns columns w + NW q.  No smem traffic in the sweep.
//  * The sweeps are dgetrf + dgetrs' own: step j of the factorization finds the
//    pivot, scales the multipliers (x * (1/pivot), dgetf2) and applies the rank-1
//    update to the trailing columns AND to the right-hand side (that is the L
//    solve, same fma order); then a backward sweep x_k = w_k * (1/u_kk) (OpenBLAS'
//    trsm kernels multiply by the inverted diagonal), w_i -= u_ik x_k (k
//    descending) solves with U.  Pivot sequence, U diagonal
//    (the singularity test) and the solve order are LAPACK's.
//  * Interchanges move nothing: each row keeps its physical place and carries
//    its LAPACK *position*; the argmax breaks ties on position (idamax's first
//    index of the permuted column), and the position bookkeeping reproduces the
//    swap of rows j and p.
//  * One __syncthreads per column and sweep: warp (j mod NW) owns column j, finds
//    the pivot (REDUX argmax), writes the multipliers of all rows to a double-
//    buffered smem vector; every warp then broadcasts the pivot row by shuffles
//    and updates its own columns right of j (backward: the RHS columns).
//  * rt^ streams into smem by cp.async while the sweep runs; out = r - rt * W
//    is DMMA (mma.sync m16n8k4 f64 -> SASS DMMA.8x8x4) from smem.
#include <climits>

#include "bri_common.cuh"
#include "bri_internal.h"

namespace bri {

namespace {

// warps per CTA: 8 up to N = 64 (the 64 x 128 augmented block is 32 doubles per lane);
// 16 for N = 96 so that a lane's share (36 doubles) stays in registers
#ifndef BRI_SN_WARPS_SMALL
#define BRI_SN_WARPS_SMALL 8
#endif
#ifndef BRI_SN_WARPS_96
#define BRI_SN_WARPS_96 16
#endif
template <int N>
constexpr int sn_warps() { return N > 64 ? BRI_SN_WARPS_96 : BRI_SN_WARPS_SMALL; }

// named barriers (ids 1, 2; 0 is __syncthreads): the producer warp of a step arrives,
// the others sync — the producer does not wait for its own publication
BRI_DEVI void bar_arrive(int id, int nthreads) {
  asm volatile("barrier.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
BRI_DEVI void bar_sync(int id, int nthreads) {
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

BRI_DEVI void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
BRI_DEVI void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
BRI_DEVI void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int N>
constexpr int sn_ldr() { return N + 8; }   // == 8 (mod 16) doubles: conflict-free DMMA fragment loads

template <int N>
constexpr int small_smem() { return 2 * N * sn_ldr<N>() * 8; }

#ifdef BRI_SMALL_PROFILE
__device__ unsigned long long g_small_phase[8];
#define SPROF(k)                                                   \
  do {                                                             \
    if (threadIdx.x == 0 && blockIdx.x == 0) {                     \
      const unsigned long long now = clock64();                    \
      atomicAdd(&g_small_phase[k], now - t_last);                  \
      t_last = now;                                                \
    }                                                              \
  } while (0)
#else
#define SPROF(k) do { } while (0)
#endif

// mode 0: Schur node (items: p, rt, l, r, out);  mode 1: out = p^-1 (items: in, -, -, -, out)
//
// BLK (opt-in, BRI_SMALL_BLOCKED=1): the columns are dealt to the warps in BLOCKS (warp w owns matrix and right-hand-
// side columns [w * QM, (w + 1) * QM)), and a warp factors its whole QM-column panel by itself —
// pivot search, multipliers and the panel's own rank-1 updates all inside one warp, no CTA barrier
// and no shared-memory round trip per column — then publishes the panel's QM multiplier columns
// once (one named barrier per PANEL instead of per column).  The other warps apply the panel to
// their columns step by step (same fma(-l_ij, u_jc, a_ic), same j order: results are bit-identical
// to the column-cyclic schedule); the owner of the next panel updates its matrix columns first,
// factors and publishes, and only then catches up on its right-hand-side columns, so the critical
// path is the chain of panel factorizations.  Measured (tools/bench_small.sh): bit-identical outputs
// and the same time per launch as the default column-cyclic schedule (!BLK: one barrier per column,
// owner of column j + 1 looks ahead) — 60.0 vs 60.2 us at N = 64 — so the per-column cost is not
// the barrier protocol but the dependent chain of a pivot step itself.
template <int N, bool BLK>
__global__ void __launch_bounds__(32 * sn_warps<N>(), 1) small_node_kernel(ArenaView a, const int* items, int mode,
                                                                         int* status) {
  constexpr int NW = sn_warps<N>();
  constexpr int SN_THREADS = 32 * NW;
  constexpr int R = N / 32;        // rows per lane
  constexpr int Q = 2 * N / NW;    // augmented columns per warp (N of p^, N of the right-hand side)
  constexpr int QM = Q / 2;        // matrix columns per warp
  constexpr int LDR = sn_ldr<N>();
  extern __shared__ double sm[];
  double* RTs = sm;                // RTs[k * LDR + i] = rt^(i, k)
  double* Ws = sm + N * LDR;       // Ws[k * LDR + c]  = W(k, c)
  __shared__ double mult[2][N];
  __shared__ double pvs[N];
  __shared__ int prow_s[2], ppos_s[2];
  __shared__ unsigned long long scale_bits;
  __shared__ int first_bad;

  const int n = a.n, ld = a.ld;
  const int* it = items + 5 * blockIdx.x;
  const double* P = a.base + (long long)it[0] * a.slot_elems;
  const double* Rt = a.base + (long long)it[1] * a.slot_elems;
  const double* Lb = a.base + (long long)it[2] * a.slot_elems;
  const double* Rb = a.base + (long long)it[3] * a.slot_elems;
  double* Out = a.base + (long long)it[4] * a.slot_elems;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // augmented column held in register column q: matrix columns are < N, right-hand side N + c
  auto colof = [&](int q) {
    return BLK ? (q < QM ? warp * QM + q : N + warp * QM + (q - QM)) : warp + NW * q;
  };
#ifdef BRI_SMALL_PROFILE
  unsigned long long t_last = clock64();
#endif

  if (tid == 0) {
    scale_bits = 0ull;
    first_bad = INT_MAX;
  }
  // rt^ -> smem, asynchronously (only the GEMM reads it); rows k >= n are zero
  if (mode == 0) {
    for (int e = tid; e < N * (N / 2); e += SN_THREADS) {
      const int k = e / (N / 2), i2 = 2 * (e % (N / 2));
      double* dst = RTs + k * LDR + i2;
      if (k < n && i2 < n) cp_async16(dst, Rt + i2 + (long long)k * ld);
      else dst[0] = dst[1] = 0.0;
    }
    cp_async_commit();
    for (int e = tid; e < (N - n) * N; e += SN_THREADS) Ws[(n + e / N) * LDR + e % N] = 0.0;
  }

  // [p^ | l^] (or [p^ | I]) into registers; max |p| for the singularity test
  double A[R][Q];
  int pos[R];
  double mx = 0.0;
#pragma unroll
  for (int h = 0; h < R; ++h) {
    const int r = lane + 32 * h;
    pos[h] = r;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int c = colof(q);
      double v = 0.0;
      if (c < N) {
        if (r < n && c < n) v = P[r + (long long)c * ld];
        const double av = fabs(v);
        if (__double_as_longlong(av) > __double_as_longlong(mx)) mx = av;   // NaN counts as largest
      } else if (r < n && c - N < n) {
        v = mode == 1 ? (r == c - N ? 1.0 : 0.0) : Lb[r + (long long)(c - N) * ld];
      }
      A[h][q] = v;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double o = __shfl_xor_sync(0xffffffffu, mx, off);
    if (__double_as_longlong(o) > __double_as_longlong(mx)) mx = o;
  }
  __syncthreads();
  if (lane == 0) atomicMax(&scale_bits, (unsigned long long)__double_as_longlong(mx));

  SPROF(0);
  // ------------------------------------------------ LU + forward sweep, one barrier per column
  // Pivot step for column jn held in register column qn by the calling warp: argmax
  // |x| over rows at positions >= jn (ties -> smallest position, NaN never wins), the
  // signed pivot, dgetf2's multipliers x * (1/pivot) of the rows below (kept in place
  // as L(i, jn) and published to smem for every warp), the pivot row and position.
  auto pivot_step = [&](int jn, int qn) {
    const int bufn = jn & 1;
    double bv = -1.0;
    int bi = INT_MAX;
#pragma unroll
    for (int h = 0; h < R; ++h) {
      const int r = lane + 32 * h;
      const double av = fabs(A[h][qn]);
      if (r < n && pos[h] >= jn && (av > bv || (av == bv && pos[h] < bi))) {
        bv = av;
        bi = pos[h];
      }
    }
#if defined(BRI_SN_SKIP) && (BRI_SN_SKIP & 1)
    bi = jn;               // experiment: no pivot search (timing only)
#else
    warp_argmax_fast(bv, bi);
#endif
    const int pp = (bi == INT_MAX) ? jn : bi;   // all NaN: pivot in place
    int oh = -1;
#pragma unroll
    for (int h = 0; h < R; ++h)
      if (lane + 32 * h < n && pos[h] == pp) oh = h;
    double mine = 0.0;
#pragma unroll
    for (int h = 0; h < R; ++h)
      if (oh == h) mine = A[h][qn];
    const unsigned m = __ballot_sync(0xffffffffu, oh >= 0);
    const int src = __ffs(m) - 1;
    const double pv = __shfl_sync(0xffffffffu, mine, src);
    const int rp = __shfl_sync(0xffffffffu, lane + 32 * (oh < 0 ? 0 : oh), src);
    const bool recip = fabs(pv) >= kSfmin;
#if defined(BRI_SN_SKIP) && (BRI_SN_SKIP & 2)
    const double rinv = pv;   // experiment: no reciprocal (timing only)
#else
    const double rinv = 1.0 / pv;
#endif
#pragma unroll
    for (int h = 0; h < R; ++h) {
      const int r = lane + 32 * h;
      double l = 0.0;
      if (r < n && pos[h] >= jn && r != rp && pv != 0.0) {
        l = recip ? A[h][qn] * rinv : A[h][qn] / pv;
        A[h][qn] = l;
      }
      mult[bufn][r] = l;
    }
    if (lane == 0) {
      prow_s[bufn] = rp;
      ppos_s[bufn] = pp;
      pvs[jn] = pv;
    }
  };
  // column q of this warp for step j: a_iq -= l_i * u_jq (u_jq from the pivot row's lane)
  auto update_col = [&](int q, const double (&lm)[R], int srcl, int hp) {
    double mine = A[0][q];
#pragma unroll
    for (int h = 1; h < R; ++h) mine = (hp == h) ? A[h][q] : mine;
    const double u = __shfl_sync(0xffffffffu, mine, srcl);
#pragma unroll
    for (int h = 0; h < R; ++h) A[h][q] = fma(-lm[h], u, A[h][q]);   // l = 0: unchanged
  };
  // make the max |p| reduction and the zeroed smem visible before the sweep
  __syncthreads();
  if constexpr (BLK) {
    __shared__ double bmult[3][QM][N];   // a panel's multiplier columns, by physical row (3 panels in flight)
    __shared__ int prow_b[N], ppos_b[N];
    // Factor this warp's panel pw (register columns 0 .. QM-1, steps j = pw * QM + jq): dgetf2
    // inside one warp.  Per step: argmax |x| over the rows at positions >= j (ties -> smallest
    // position, NaN never wins), multipliers x * (1/pivot) kept in place and published, the
    // position bookkeeping of the interchange, and the rank-1 update of the panel's own columns
    // right of j.
    auto factor_panel = [&](int pw) {
      double(*bm)[N] = bmult[pw % 3];
#pragma unroll
      for (int jq = 0; jq < QM; ++jq) {
        const int j = pw * QM + jq;
        if (j >= n) break;
        double bv = -1.0;
        int bi = INT_MAX;
#pragma unroll
        for (int h = 0; h < R; ++h) {
          const int r = lane + 32 * h;
          const double av = fabs(A[h][jq]);
          if (r < n && pos[h] >= j && (av > bv || (av == bv && pos[h] < bi))) {
            bv = av;
            bi = pos[h];
          }
        }
        warp_argmax_fast(bv, bi);
        const int pp = (bi == INT_MAX) ? j : bi;   // all NaN: pivot in place
        int oh = -1;
#pragma unroll
        for (int h = 0; h < R; ++h)
          if (lane + 32 * h < n && pos[h] == pp) oh = h;
        double mine = 0.0;
#pragma unroll
        for (int h = 0; h < R; ++h)
          if (oh == h) mine = A[h][jq];
        const unsigned m = __ballot_sync(0xffffffffu, oh >= 0);
        const int src = __ffs(m) - 1;
        const double pv = __shfl_sync(0xffffffffu, mine, src);
        const int rp = __shfl_sync(0xffffffffu, lane + 32 * (oh < 0 ? 0 : oh), src);
        const bool recip = fabs(pv) >= kSfmin;
        const double rinv = 1.0 / pv;
        double lm[R];
#pragma unroll
        for (int h = 0; h < R; ++h) {
          const int r = lane + 32 * h;
          double l = 0.0;
          if (r < n && pos[h] >= j && r != rp && pv != 0.0) {
            l = recip ? A[h][jq] * rinv : A[h][jq] / pv;
            A[h][jq] = l;
          }
          lm[h] = l;
          bm[jq][r] = l;
        }
        if (lane == 0) {
          prow_b[j] = rp;
          ppos_b[j] = pp;
          pvs[j] = pv;
        }
#pragma unroll
        for (int h = 0; h < R; ++h) {
          if (pos[h] == j) pos[h] = pp;           // the row at position j takes the pivot's place
          else if (lane + 32 * h == rp) pos[h] = j;
        }
        const int srcl = rp & 31, hp = rp >> 5;
#pragma unroll
        for (int q = jq + 1; q < QM; ++q) update_col(q, lm, srcl, hp);
      }
    };
    // Apply the published panel pw to this warp's columns, one pivot step at a time.
    auto apply_panel = [&](int pw, bool do_pos, bool do_mat, bool do_rhs) {
      double(*bm)[N] = bmult[pw % 3];
#pragma unroll
      for (int jq = 0; jq < QM; ++jq) {
        const int j = pw * QM + jq;
        if (j >= n) break;
        const int rp = prow_b[j], pp = ppos_b[j];
        const int srcl = rp & 31, hp = rp >> 5;
        double lm[R];
#pragma unroll
        for (int h = 0; h < R; ++h) lm[h] = bm[jq][lane + 32 * h];
        if (do_pos) {
#pragma unroll
          for (int h = 0; h < R; ++h) {
            if (pos[h] == j) pos[h] = pp;
            else if (lane + 32 * h == rp) pos[h] = j;
          }
        }
        if (do_mat) {
#pragma unroll
          for (int q = 0; q < QM; ++q) update_col(q, lm, srcl, hp);
        }
        if (do_rhs) {
#pragma unroll
          for (int q = QM; q < Q; ++q) update_col(q, lm, srcl, hp);
        }
      }
    };
    if (warp == 0 && n > 0) {
      factor_panel(0);
      __syncwarp();
      bar_arrive(1, SN_THREADS);
    }
#pragma unroll 1
    for (int pw = 0; pw < NW; ++pw) {
      if (pw * QM >= n) break;
      const bool owner = (warp == pw);
      if (!owner) bar_sync(1 + (pw & 1), SN_THREADS);   // panel pw is published
      if (warp == pw + 1 && (pw + 1) * QM < n) {
        apply_panel(pw, true, true, false);
        factor_panel(pw + 1);
        __syncwarp();
        bar_arrive(1 + ((pw + 1) & 1), SN_THREADS);
        apply_panel(pw, false, false, true);
      } else {
        apply_panel(pw, !owner, warp > pw, true);
      }
    }
  } else {
  if (warp == 0 && n > 0) {
    pivot_step(0, 0);
    bar_arrive(1, SN_THREADS);
  }
  // qj (the register column of j) must be a compile-time index: unrolled outer loop over
  // register columns, rolled inner loop over the warps that own them.  Lookahead: the
  // owner of column j+1 updates that column first, publishes step j+1's pivot and ARRIVES
  // at that step's named barrier (ids alternate 1 / 2) before its other columns; the other
  // warps sync on it.  The critical path per column is one pivot search, not a full update.
#pragma unroll
  for (int qj = 0; qj < N / NW; ++qj)
#pragma unroll 1
  for (int wj = 0; wj < NW; ++wj) {
    const int j = qj * NW + wj;
    if (j >= n) break;
    const int buf = j & 1;
    if (warp != wj) bar_sync(1 + buf, SN_THREADS);   // the owner of column j published it
    const int rp = prow_s[buf], pp = ppos_s[buf];
    const int srcl = rp & 31, hp = rp >> 5;
    double lm[R];
#pragma unroll
    for (int h = 0; h < R; ++h) lm[h] = mult[buf][lane + 32 * h];
#pragma unroll
    for (int h = 0; h < R; ++h) {
      if (pos[h] == j) pos[h] = pp;           // the row at position j takes the pivot's place
      else if (lane + 32 * h == rp) pos[h] = j;
    }
    const bool wrap = (wj == NW - 1);         // column j+1 sits in the next register column
    const bool la = (j + 1 < n) && warp == (wrap ? 0 : wj + 1);
    if (la) {
      if (!wrap) {
        update_col(qj, lm, srcl, hp);
        pivot_step(j + 1, qj);
      } else if (qj + 1 < N / NW) {
        update_col(qj + 1, lm, srcl, hp);
        pivot_step(j + 1, qj + 1);
      }
      bar_arrive(1 + ((j + 1) & 1), SN_THREADS);
    }
    // rank-1 update of the trailing matrix and the forward sweep of the right-hand side
    // (dgetrs' L solve applies the same fma(-l_ij, w_j, w_i) in the same j order); register
    // columns left of qj are dead for every warp (compile-time), column qj is live only right
    // of j, and the lookahead column is already done
#if defined(BRI_SN_SKIP) && (BRI_SN_SKIP & 4)
    if (false)             // experiment: no trailing updates (timing only)
#endif
#pragma unroll
    for (int q = qj; q < Q; ++q) {
      const int c = warp + NW * q;
      const bool done = (la && c == j + 1);
      if (q == qj || q == qj + 1) {
        if (c > j && !done) update_col(q, lm, srcl, hp);
      } else {
        update_col(q, lm, srcl, hp);
      }
    }
  }

  }   // !BLK

  SPROF(1);
  // ------------------------------------------------ backward sweep (dgetrs' U solve), no barriers
  //   x_k = w_k * (1/u_kk);  w_i -= u_ik x_k  (i < k),  k descending.  U is static by now:
  //   its columns go to smem once (the owner of column k writes U(., k) by physical row),
  //   and every warp then solves its own right-hand-side columns independently.
  {
    __shared__ int row_at[N];
    __shared__ double rpv[N];   // 1 / u_kk, one division per pivot in parallel (was one per step on every warp's chain)
    double* Us = Ws;   // U(r, k) at Us[k * LDR + r] (physical row r); Ws is rebuilt afterwards
    __syncthreads();
#pragma unroll
    for (int h = 0; h < R; ++h) {
      const int r = lane + 32 * h;
      if (warp == 0 && r < n) row_at[pos[h]] = r;
#pragma unroll
      for (int q = 0; q < Q / 2; ++q) {      // matrix columns of this warp
        const int c = colof(q);
        if (c < n && r < N) Us[c * LDR + r] = (r < n && pos[h] < c) ? A[h][q] : 0.0;
      }
    }
    for (int k = tid; k < n; k += SN_THREADS) rpv[k] = 1.0 / pvs[k];
    __syncthreads();
    for (int k = n - 1; k >= 0; --k) {
      const int rk = row_at[k];
      const int srcl = rk & 31, hk = rk >> 5;
      const double rkk = rpv[k];
      double um[R];
#pragma unroll
      for (int h = 0; h < R; ++h) um[h] = Us[k * LDR + lane + 32 * h];
#pragma unroll
      for (int q = Q / 2; q < Q; ++q) {       // right-hand-side columns only
        double mine = A[0][q];
#pragma unroll
        for (int h = 1; h < R; ++h) mine = (hk == h) ? A[h][q] : mine;
        const double x = __shfl_sync(0xffffffffu, mine, srcl) * rkk;
#pragma unroll
        for (int h = 0; h < R; ++h) A[h][q] = (lane + 32 * h == rk) ? x : fma(-um[h], x, A[h][q]);
      }
    }
  }

  // ------------------------------------------------ singularity test (U diagonal = the pivots)
  __syncthreads();
  SPROF(2);
  {
    const double tol = (double)n * kEps * __longlong_as_double((long long)scale_bits);
    for (int i = tid; i < n; i += SN_THREADS)
      if (!(fabs(pvs[i]) > tol)) atomicMin(&first_bad, i);
  }

  // ------------------------------------------------ W(k, :) = the solved row at position k
#pragma unroll
  for (int h = 0; h < R; ++h) {
    const int r = lane + 32 * h;
    if (r < n) {
      const int k = pos[h];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int c = colof(q) - N;
        if (c >= 0 && c < n) {
          const double x = A[h][q];
          if (mode == 1) Out[k + (long long)c * ld] = x;
          else Ws[k * LDR + c] = x;
        }
      }
      if (mode == 0)
        for (int c = n; c < N; ++c) Ws[k * LDR + c] = 0.0;
    }
  }
  __syncthreads();
  if (tid == 0 && status != nullptr) status[blockIdx.x] = first_bad == INT_MAX ? 0 : first_bad + 1;
  SPROF(3);
  if (mode == 1) return;

  // ------------------------------------------------ out = r - rt * W on the tensor cores
  cp_async_wait_all();
  __syncthreads();
  SPROF(4);
  constexpr int MT = N / 16, NT = N / 8;
  const int g = lane >> 2, t = lane & 3;
  const int kmax = (n + 3) & ~3;
  for (int tt = warp; tt < MT * NT; tt += NW) {
    const int i0 = 16 * (tt % MT), c0 = 8 * (tt / MT);
    if (i0 >= n || c0 >= n) continue;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k0 = 0; k0 < kmax; k0 += 4) {
      const double* ra = RTs + (k0 + t) * LDR + i0 + g;
      dmma_16x8x4(acc, ra[0], ra[8], Ws[(k0 + t) * LDR + c0 + g]);
    }
    const int i = i0 + g, c = c0 + 2 * t;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int ii = i + (v >> 1) * 8, cc = c + (v & 1);
      if (ii < n && cc < n) {
        const long long off = ii + (long long)cc * ld;
        Out[off] = Rb[off] - acc[v];
      }
    }
  }
  SPROF(5);
}

int g_small_blocked = -1;   // -1: BRI_SMALL_BLOCKED (default 0: measured equal at N = 32 / 64, 4% slower at N = 96)

bool small_blocked() {
  if (g_small_blocked < 0) {
    const char* e = getenv("BRI_SMALL_BLOCKED");
    g_small_blocked = (e != nullptr && e[0] == '1') ? 1 : 0;
  }
  return g_small_blocked != 0;
}

template <int N>
cudaError_t launch_small_t(const ArenaView& a, const int* items, int count, int mode, int* status,
                           cudaStream_t s) {
  count_launch();
  if (small_blocked())
    small_node_kernel<N, true><<<count, 32 * sn_warps<N>(), small_smem<N>(), s>>>(a, items, mode, status);
  else
    small_node_kernel<N, false><<<count, 32 * sn_warps<N>(), small_smem<N>(), s>>>(a, items, mode, status);
  return cudaGetLastError();
}

}  // namespace

#ifdef BRI_SMALL_PROFILE
void small_profile_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_small_phase, sizeof(g_small_phase));
  unsigned long long z[8] = {0};
  cudaMemcpyToSymbol(g_small_phase, z, sizeof(z));
}
#endif

void small_set_blocked(int on) { g_small_blocked = on ? 1 : 0; }   // tools: switch schedules in one process

cudaError_t configure_small() {
  cudaError_t e = cudaSuccess;
  auto set = [&](const void* f, int bytes) {
    if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  };
  set((const void*)small_node_kernel<32, true>, small_smem<32>());
  set((const void*)small_node_kernel<32, false>, small_smem<32>());
  set((const void*)small_node_kernel<64, true>, small_smem<64>());
  set((const void*)small_node_kernel<64, false>, small_smem<64>());
  set((const void*)small_node_kernel<SMALL_MAX, true>, small_smem<SMALL_MAX>());
  set((const void*)small_node_kernel<SMALL_MAX, false>, small_smem<SMALL_MAX>());
  return e;
}

cudaError_t launch_small_node(const ArenaView& a, const int* items, int count, int mode,
                              int* status, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  if (a.n <= 32) return launch_small_t<32>(a, items, count, mode, status, s);
  if (a.n <= 64) return launch_small_t<64>(a, items, count, mode, status, s);
  if (a.n <= SMALL_MAX) return launch_small_t<SMALL_MAX>(a, items, count, mode, status, s);
  return cudaErrorInvalidValue;
}

}  // namespace bri
