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

// ---------------------------------------------------------------------------
// Seeded Gaussian test matrices generated blockwise on the device (BASELINE
// config 5: M = G + m I, G i.i.d. N(0, 1) "generated blockwise from seed 4";
// the reference has no blockwise scheme).
//
//   element (r, c), 0-based over order m:  e = r * m + c
//   (o0, o1, o2, o3) = Philox4x64-10(counter = (e / 4, 0, 0, 0), key = (seed, 0))
//     — numpy's np.random.Philox bit generator (Random123), restated here
//   pair q = (e % 4) / 2:  u1 = ((o_{2q} >> 11) + 1) 2^-53 in (0, 1],
//                          u2 = (o_{2q+1} >> 11) 2^-53 in [0, 1)
//   Box-Muller: rho = sqrt(-2 log u1), theta = 2 pi u2,
//               g = rho cos(theta) for even e, rho sin(theta) for odd e
//   M_rc = g + (r == c ? shift : 0)
//
// Every element depends only on (seed, m, r, c), so any block (or any padded
// window view) is produced independently and the matrix does not depend on
// the partition k.  The integer stream is exact; log/sin/cos are CUDA's
// (within 1-2 ulp of glibc's, which the numpy restatement uses).
// ---------------------------------------------------------------------------
namespace bri {
namespace {

__device__ __forceinline__ void philox4x64_10(unsigned long long c[4], unsigned long long k0,
                                              unsigned long long k1) {
  const unsigned long long M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
  const unsigned long long W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    const unsigned long long hi0 = __umul64hi(M0, c[0]), lo0 = M0 * c[0];
    const unsigned long long hi1 = __umul64hi(M1, c[2]), lo1 = M1 * c[2];
    const unsigned long long n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += W0;
    k1 += W1;
  }
}

struct RandnParams {
  long long m;
  unsigned long long seed;
  double shift;
  const int* rmap;  // view index -> global index (nullptr: identity)
  const int* cmap;
};

__device__ __forceinline__ double randn_element(const RandnParams& p, long long r, long long c) {
  if (r >= p.m || c >= p.m) return r == c ? 1.0 : 0.0;  // identity padding [[M, 0], [0, I]]
  const unsigned long long e = (unsigned long long)r * (unsigned long long)p.m + (unsigned long long)c;
  unsigned long long ctr[4] = {e >> 2, 0ULL, 0ULL, 0ULL};
  philox4x64_10(ctr, p.seed, 0ULL);
  const int q = (int)(e & 3ULL) >> 1;
  const unsigned long long a = q ? ctr[2] : ctr[0], bb = q ? ctr[3] : ctr[1];
  const double u1 = __dmul_rn((double)((a >> 11) + 1ULL), 0x1.0p-53);
  const double u2 = __dmul_rn((double)(bb >> 11), 0x1.0p-53);
  const double rho = __dsqrt_rn(__dmul_rn(-2.0, log(u1)));
  const double theta = __dmul_rn(6.283185307179586, u2);
  const double g = __dmul_rn(rho, (e & 1ULL) ? sin(theta) : cos(theta));
  return r == c ? __dadd_rn(g, p.shift) : g;
}

// grid.y = item; each CTA strides over the block's rows x cols elements.
__global__ void __launch_bounds__(256) randn_kernel(RandnParams p, double* base, long long slot_elems, int ld,
                                                    int rows, int cols, long long row0, long long col0,
                                                    const int* items) {
  double* out = base;
  long long r0 = row0, c0 = col0;
  if (items != nullptr) {
    const int* it = items + 3 * blockIdx.y;
    r0 = (long long)it[0] * rows;
    c0 = (long long)it[1] * cols;
    out = base + (long long)it[2] * slot_elems;
  }
  const long long total = (long long)rows * cols;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(idx / cols), c = (int)(idx % cols);
    const long long vr = r0 + r, vc = c0 + c;
    const long long gr = p.rmap != nullptr ? (long long)p.rmap[vr] : vr;
    const long long gc = p.cmap != nullptr ? (long long)p.cmap[vc] : vc;
    out[(long long)r * ld + c] = randn_element(p, gr, gc);
  }
}

}  // namespace

cudaError_t launch_randn(const RandnArgs& g, double* base, long long slot_elems, int ld, int rows, int cols,
                         long long row0, long long col0, const int* items, int count, cudaStream_t s) {
  if (count > 65535 || rows < 1 || cols < 1) return cudaErrorInvalidValue;
  RandnParams p{g.m, g.seed, g.shift, g.rmap, g.cmap};
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long total = (long long)rows * cols;
  long long want = (total + 255) / 256;
  const long long cap = (long long)sms * 8 / (count > 0 ? count : 1) + 1;
  const unsigned gx = (unsigned)(want < cap ? want : cap);
  count_launch();
  randn_kernel<<<dim3(gx, count), 256, 0, s>>>(p, base, slot_elems, ld, rows, cols, row0, col0, items);
  return cudaGetLastError();
}

}  // namespace bri
