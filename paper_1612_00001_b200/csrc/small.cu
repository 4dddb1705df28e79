// K6: fused one-CTA Schur node / block inverse for small blocks (n <= 96), sm_100a.
//
// For b <= 96 a whole node of the reference's `_fold` (engine.py:157-180) fits
// in one SM's shared memory: pivot LU with partial pivoting (dgetrf semantics
// on the X-world view, core.py:249), the growth-scaled singularity test
// (core.py:200-209), the solve W = P^-1 * l (dgetrs, core.py:259) and the
// fused update out = r - rt * W run in one launch per DAG level, one CTA per
// node.  This is the latency-bound regime of BASELINE config 1 (b = 64) and
// of every small-b case in the reference's own test-suite.
//
// In X-world the node computes  out^ = r^ - rt^ * (p^)^-1 * l^  which is the
// transpose of the reference's  r - l @ (inv(p) @ rt)  (all hats are the
// column-major views of the row-major blocks).
#include <climits>

#include "bri_common.cuh"
#include "bri_internal.h"

namespace bri {

namespace {

constexpr int SN_THREADS = 256;

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

template <int NMAX>
__global__ void __launch_bounds__(SN_THREADS) small_node_kernel(ArenaView a, const int* items, int mode,
                                                                int* status) {
  constexpr int LDS = NMAX + 1;
  constexpr int LDW = NMAX + 8;    // W rows: 8 columns x 4 rows per warp access hit 2 wavefronts
  extern __shared__ double sm[];
  double* F = sm;                  // factor of p^   (F[c * LDS + i] = element (i, c))
  double* RT = F + NMAX * LDS;     // rt^ (mode 0 only)
  double* W = RT + NMAX * LDS;     // right-hand side / solution, row-major: W[i * LDW + c]
  __shared__ int perm[NMAX];
  __shared__ int piv_s;
  __shared__ unsigned long long scale_bits;
  __shared__ int first_bad;

  const int n = a.n, ld = a.ld;
  const int* it = items + 5 * blockIdx.x;
  const double* P = a.base + (long long)it[0] * a.slot_elems;
  const double* Rt = a.base + (long long)it[1] * a.slot_elems;
  const double* Lb = a.base + (long long)it[2] * a.slot_elems;
  const double* R = a.base + (long long)it[3] * a.slot_elems;
  double* Out = a.base + (long long)it[4] * a.slot_elems;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

#ifdef BRI_SMALL_PROFILE
  unsigned long long t_last = clock64();
#endif
  if (tid == 0) {
    scale_bits = 0ull;
    first_bad = INT_MAX;
  }
  if (tid < n) perm[tid] = tid;
  __syncthreads();
  double mx = 0.0;
  for (int e = tid; e < n * n; e += SN_THREADS) {
    const int i = e % n, c = e / n;
    const double v = P[i + (long long)c * ld];
    F[c * LDS + i] = v;
    const double av = fabs(v);
    if (__double_as_longlong(av) > __double_as_longlong(mx)) mx = av;
    if (mode == 0) RT[c * LDS + i] = Rt[i + (long long)c * ld];
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double o = __shfl_xor_sync(0xffffffffu, mx, off);
    if (__double_as_longlong(o) > __double_as_longlong(mx)) mx = o;
  }
  if (lane == 0) atomicMax(&scale_bits, (unsigned long long)__double_as_longlong(mx));
  __syncthreads();

  SPROF(0);
  // ------------------------------------------------ dgetf2 on F (in smem)
  for (int j = 0; j < n; ++j) {
    if (warp == 0) {
      double bv = -1.0;
      int bi = INT_MAX;
      for (int i = j + lane; i < n; i += 32) argmax_merge(bv, bi, fabs(F[j * LDS + i]), i);
      warp_argmax(bv, bi);
      if (lane == 0) piv_s = (bi == INT_MAX) ? j : bi;
    }
    __syncthreads();
    const int p = piv_s;
    const double pv = F[j * LDS + p];
    if (p != j && pv != 0.0) {
      for (int c = tid; c < n; c += SN_THREADS) {
        const double t = F[c * LDS + j];
        F[c * LDS + j] = F[c * LDS + p];
        F[c * LDS + p] = t;
      }
      if (tid == 0) {
        const int t = perm[j];
        perm[j] = perm[p];
        perm[p] = t;
      }
    }
    __syncthreads();
    const double piv = F[j * LDS + j];
    if (piv != 0.0) {
      const bool recip = fabs(piv) >= kSfmin;
      const double rinv = 1.0 / piv;
      for (int i = j + 1 + tid; i < n; i += SN_THREADS) {
        const double x = F[j * LDS + i];
        F[j * LDS + i] = recip ? x * rinv : x / piv;
      }
    }
    __syncthreads();
    // rank-1 update, one warp per column (no index division, coalesced rows)
    for (int c = j + 1 + warp; c < n; c += SN_THREADS / 32) {
      const double u = F[c * LDS + j];
      for (int i = j + 1 + lane; i < n; i += 32) F[c * LDS + i] = fma(-F[j * LDS + i], u, F[c * LDS + i]);
    }
    __syncthreads();
  }

  SPROF(1);
  // ------------------------------------------------ singularity test
  {
    const double tol = (double)n * kEps * __longlong_as_double((long long)scale_bits);
    for (int i = tid; i < n; i += SN_THREADS)
      if (!(fabs(F[i * LDS + i]) > tol)) atomicMin(&first_bad, i);
    __syncthreads();
    if (tid == 0 && status != nullptr) status[blockIdx.x] = first_bad == INT_MAX ? 0 : first_bad + 1;
  }

  // ------------------------------------------------ W = P * rhs, then L, U solves
  for (int e = tid; e < n * n; e += SN_THREADS) {
    const int x = e % n, c = e / n;
    const int s = perm[x];
    W[x * LDW + c] = (mode == 1) ? (s == c ? 1.0 : 0.0) : Lb[s + (long long)c * ld];
  }
  __syncthreads();
  SPROF(2);
  // Forward (unit L) and backward (U) substitution, TPC threads per right-hand
  // side column (one warp holds 32 / TPC columns): each step's row updates are
  // split between them and a __syncwarp orders the steps.  Every element sees
  // the column-serial operation sequence (fma(-x_k, L_ik, w_i) for k ascending;
  // x_k = w_k / U_kk, then fma(-x_k, U_ik, w_i) for k descending).
  {
    constexpr int TPC = (SN_THREADS / NMAX) >= 8 ? 8 : (SN_THREADS / NMAX) >= 4 ? 4 : 2;
    const int c = tid / TPC, part = tid % TPC;
    double* w = W + c;               // element i of this column at w[i * LDW]
    const bool col = c < n;
    for (int k = 0; k < n; ++k) {
      if (col) {
        const double xk = w[k * LDW];
        for (int i = k + 1 + part; i < n; i += TPC) w[i * LDW] = fma(-xk, F[k * LDS + i], w[i * LDW]);
      }
      __syncwarp();
    }
    for (int k = n - 1; k >= 0; --k) {
      double xk = 0.0;
      if (col) xk = w[k * LDW] / F[k * LDS + k];
      __syncwarp();
      if (col) {
        if (part == 0) w[k * LDW] = xk;
        for (int i = part; i < k; i += TPC) w[i * LDW] = fma(-xk, F[k * LDS + i], w[i * LDW]);
      }
      __syncwarp();
    }
  }
  __syncthreads();

  SPROF(3);
  if (mode == 1) {
    for (int e = tid; e < n * n; e += SN_THREADS) {
      const int i = e % n, c = e / n;
      Out[i + (long long)c * ld] = W[i * LDW + c];
    }
    return;
  }

  // ------------------------------------------------ out = r - rt * W
  const int tiles = (n + 3) / 4;
  for (int tt = tid; tt < tiles * tiles; tt += SN_THREADS) {
    const int i0 = (tt % tiles) * 4, c0 = (tt / tiles) * 4;
    double acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
    for (int k = 0; k < n; ++k) {
      double ra[4], wb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) ra[u] = (i0 + u < n) ? RT[k * LDS + i0 + u] : 0.0;
#pragma unroll
      for (int v = 0; v < 4; ++v) wb[v] = (c0 + v < n) ? W[k * LDW + c0 + v] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(ra[u], wb[v], acc[u][v]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int i = i0 + u, c = c0 + v;
        if (i < n && c < n) {
          const long long off = i + (long long)c * ld;
          Out[off] = R[off] - acc[u][v];
        }
      }
  }
  SPROF(4);
}

template <int NMAX>
constexpr int small_smem() { return (2 * NMAX * (NMAX + 1) + NMAX * (NMAX + 8)) * 8; }

template <int NMAX>
cudaError_t launch_small_t(const ArenaView& a, const int* items, int count, int mode, int* status,
                           cudaStream_t s) {
  const int smem = small_smem<NMAX>();
  count_launch();
  small_node_kernel<NMAX><<<count, SN_THREADS, smem, s>>>(a, items, mode, status);
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

cudaError_t configure_small() {
  cudaError_t e = cudaFuncSetAttribute(small_node_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       small_smem<32>());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(small_node_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, small_smem<64>());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(small_node_kernel<SMALL_MAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             small_smem<SMALL_MAX>());
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
