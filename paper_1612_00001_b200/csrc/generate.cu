// On-device generation of the LS-SVM kernel system matrix (reference
// providers.py:93-120 KernelSpec, 175-200 _KernelSource.rect):
//
//   element (g_r, g_c), 0-based over order m = n + 1:
//     (0, 0)                   -> 0
//     row 0 or column 0        -> 1
//     interior                 -> exp(sq / denom) + (g_r == g_c ? ridge : 0)
//        sq    = sum_t (x[g_r-1, t] - x[g_c-1, t])^2   (numpy pairwise order)
//        denom = -2 sigma^2, ridge = 1 / gamma          (computed by the caller)
//   and for padded layouts [[M, 0], [0, I]]: g >= m -> identity.
//
// Blocks are written straight into arena slots (M is never stored), or the
// whole matrix into a dense row-major buffer (kernel_matrix / verify).  The
// squared-difference sum reproduces numpy's pairwise summation (the order
// np.sum uses along a contiguous axis: <8 terms sequential, <=128 terms in 8
// interleaved accumulators, longer runs split in halves rounded down to a
// multiple of 8), with explicit round-to-nearest ops so nothing is contracted
// into an FMA: the sums are bit-identical to the reference's, only exp() may
// differ by an ulp.
#include "bri_internal.h"

namespace bri {
namespace {

constexpr int TILE = 32;
constexpr int ROWS_PER_THREAD = 4;  // 32 x 8 threads, 4 rows each
constexpr int DSTAGE = 64;          // feature counts up to this are staged in shared memory

__device__ __forceinline__ double sqdiff(const double* a, const double* b, int i) {
  const double t = __dsub_rn(a[i], b[i]);
  return __dmul_rn(t, t);
}

__device__ double pairwise_sqdist(const double* a, const double* b, int n) {
  if (n < 8) {
    double res = -0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, sqdiff(a, b, i));
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = sqdiff(a, b, j);
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], sqdiff(a, b, i + j));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, sqdiff(a, b, i));
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  const double left = pairwise_sqdist(a, b, n2);
  return __dadd_rn(left, pairwise_sqdist(a + n2, b + n2, n - n2));
}

struct RbfParams {
  const double* x;  // n x d row-major inputs
  int n, d;
  double denom, ridge;
  const int* rmap;  // view index -> global index (nullptr: identity)
  const int* cmap;
};

// One CTA per 32 x 32 tile of one output block.  items: (block row, block col,
// slot) triples (nullptr: a single dense output of order bn at `base`).
__global__ void __launch_bounds__(256) rbf_kernel(RbfParams p, double* base, long long slot_elems, int ld,
                                                  int bn, int tiles_x, const int* items) {
  __shared__ double xs[2][TILE * (DSTAGE + 1)];
  __shared__ int gidx[2][TILE];
  const int m = p.n + 1;
  int bi = 0, bj = 0;
  double* out = base;
  if (items != nullptr) {
    const int* it = items + 3 * blockIdx.y;
    bi = it[0];
    bj = it[1];
    out = base + (long long)it[2] * slot_elems;
  }
  const int r0 = (blockIdx.x / tiles_x) * TILE, c0 = (blockIdx.x % tiles_x) * TILE;
  const int tid = threadIdx.y * TILE + threadIdx.x;
  if (tid < 2 * TILE) {
    const int side = tid / TILE, t = tid % TILE;
    const int v = (side == 0 ? r0 : c0) + t;
    int g = m;  // out-of-range rows map past the matrix (never written)
    if (v < bn) {
      const long long vi = (long long)(side == 0 ? bi : bj) * bn + v;
      const int* map = side == 0 ? p.rmap : p.cmap;
      g = map != nullptr ? map[vi] : (int)vi;
    }
    gidx[side][t] = g;
  }
  __syncthreads();
  const bool staged = p.d <= DSTAGE;
  const int sd = p.d + 1;
  if (staged) {
    for (int e = tid; e < 2 * TILE * p.d; e += blockDim.x * blockDim.y) {
      const int side = e / (TILE * p.d), rem = e % (TILE * p.d), t = rem / p.d, f = rem % p.d;
      const int g = gidx[side][t];
      xs[side][t * sd + f] = (g >= 1 && g < m) ? p.x[(long long)(g - 1) * p.d + f] : 0.0;
    }
    __syncthreads();
  }
  const int c = c0 + threadIdx.x;
  const int gc = gidx[1][threadIdx.x];
  const double* xc = staged ? &xs[1][threadIdx.x * sd] : p.x + (long long)(gc - 1) * p.d;
#pragma unroll
  for (int q = 0; q < ROWS_PER_THREAD; ++q) {
    const int t = threadIdx.y + 8 * q;
    const int r = r0 + t;
    if (r >= bn || c >= bn) continue;
    const int gr = gidx[0][t];
    double v;
    if (gr >= m || gc >= m) {
      v = (gr == gc) ? 1.0 : 0.0;
    } else if (gr == 0 || gc == 0) {
      v = (gr == 0 && gc == 0) ? 0.0 : 1.0;
    } else {
      const double* xr = staged ? &xs[0][t * sd] : p.x + (long long)(gr - 1) * p.d;
      const double sq = pairwise_sqdist(xr, xc, p.d);
      v = exp(__ddiv_rn(sq, p.denom));
      if (gr == gc) v = __dadd_rn(v, p.ridge);
    }
    out[(long long)r * ld + c] = v;
  }
}

}  // namespace

cudaError_t launch_rbf(const RbfArgs& g, double* base, long long slot_elems, int ld, int bn, const int* items,
                       int count, cudaStream_t s) {
  RbfParams p{g.x, g.n, g.d, g.denom, g.ridge, g.rmap, g.cmap};
  const int tiles_x = (bn + TILE - 1) / TILE;
  const long long tiles = (long long)tiles_x * tiles_x;
  if (tiles > 0x7fffffffLL || count > 65535) return cudaErrorInvalidValue;
  count_launch();
  rbf_kernel<<<dim3((unsigned)tiles, count), dim3(TILE, 8), 0, s>>>(p, base, slot_elems, ld, bn, tiles_x, items);
  return cudaGetLastError();
}

}  // namespace bri
