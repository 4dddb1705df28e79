// K3/K4/K5: blocked LU with partial pivoting, its singularity test, the
// triangular-solve leaves and the arena copy/permute kernels, sm_100a.
//
// Replaces `invert_dense` (core.py:238-263): LAPACK dgetrf on the transposed
// (F-contiguous) view of the C-ordered block, the growth-scaled pivot test of
// `_singular_index` (core.py:200-209), then dgetrs against the right-hand side.
// In X-world (bri_common.cuh) the factorization is literally dgetrf on X, so
// pivot choices follow LAPACK (idamax: largest |x|, first index on ties).
//
// Right-looking blocked LU, panel width nb <= 32:
//   panel kernel   — one thread-block CLUSTER per matrix holds the whole
//                    (n - j0) x nb panel in distributed shared memory; per
//                    column: CTA-local argmax (warp shuffles), candidates
//                    (value, row, row contents) pushed to every CTA's smem
//                    through DSMEM, one cluster barrier, then swap + rank-1
//                    update locally.  One cluster barrier per column.
//   rowpanel kernel— applies the panel's row interchanges to every other
//                    column (as one gather through a precomputed source map,
//                    fully parallel) and solves L11 * U12 = A12 (unit lower,
//                    forward substitution) for the trailing columns.
//   GEMM (gemm.cu) — trailing update A22 -= L21 * U12.
#include <cfloat>
#include <climits>

#include "bri_common.cuh"
#include "bri_internal.h"

namespace bri {

namespace {

constexpr int MAXCS = 8;            // cluster size cap (portable)
constexpr int PANEL_THREADS = 256;

// ----------------------------------------------------------------- maxabs
__global__ void maxabs_kernel(ArenaView a, const int* slots, unsigned long long* out) {
  const int item = blockIdx.y;
  const double* x = a.base + (long long)slots[item] * a.slot_elems;
  double best = 0.0;
  const long long total = (long long)a.n * a.n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % a.n), j = (int)(e / a.n);
    const double v = fabs(x[i + (long long)j * a.ld]);
    // bit-pattern max: NaN (positive, > +Inf bits) propagates like numpy's max
    if (__double_as_longlong(v) > __double_as_longlong(best)) best = v;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double o = __shfl_xor_sync(0xffffffffu, best, off);
    if (__double_as_longlong(o) > __double_as_longlong(best)) best = o;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out + item, (unsigned long long)__double_as_longlong(best));
}

// ------------------------------------------------------------------- copy
// pairs: 2 ints per item (src slot, dst slot); copies the n x n window.
__global__ void copy_kernel(ArenaView a, const int* pairs) {
  const int item = blockIdx.y;
  const double* src = a.base + (long long)pairs[2 * item] * a.slot_elems;
  double* dst = a.base + (long long)pairs[2 * item + 1] * a.slot_elems;
  for (int j = blockIdx.x; j < a.n; j += gridDim.x)
    for (int i = threadIdx.x; i < a.n; i += blockDim.x)
      dst[i + (long long)j * a.ld] = src[i + (long long)j * a.ld];
}

// dst[x, c] = src[pi[x], c] (row gather inside every X-column; X-columns are
// contiguous memory rows so both sides stay coalesced).  identity_src: the
// source is the identity matrix (final block inversion, dgetrs against I).
__global__ void permcopy_kernel(ArenaView a, const int* pairs, const int* pi, int pi_stride,
                                int identity_src) {
  const int item = blockIdx.y;
  const double* src = a.base + (long long)pairs[2 * item] * a.slot_elems;
  double* dst = a.base + (long long)pairs[2 * item + 1] * a.slot_elems;
  const int* p = pi + (long long)item * pi_stride;
  for (int j = blockIdx.x; j < a.n; j += gridDim.x)
    for (int x = threadIdx.x; x < a.n; x += blockDim.x) {
      const int s = p[x];
      dst[x + (long long)j * a.ld] = identity_src ? (s == j ? 1.0 : 0.0) : src[s + (long long)j * a.ld];
    }
}

__global__ void pi_init_kernel(int* pi, int n) {
  const int item = blockIdx.y;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x)
    pi[(long long)item * n + x] = x;
}

// ------------------------------------------------------------------ panel
struct PanelArgs {
  ArenaView a;
  const int* slots;
  int j0, nb, rh, rhp, pidx;
  int* ipiv;
  int* sigma;
  int* pairs;
  int n_stride, pair_stride;
};

__global__ void __launch_bounds__(PANEL_THREADS) lu_panel_kernel(PanelArgs p) {
  extern __shared__ double psm[];  // nb columns x rhp rows, then rhp ints (origins)
  __shared__ double cand_val[2][MAXCS];
  __shared__ int cand_idx[2][MAXCS];
  __shared__ int cand_orig[2][MAXCS];
  __shared__ double cand_row[2][MAXCS][NBMAX];
  __shared__ double rowj[2][NBMAX];
  __shared__ int rowj_orig[2];
  __shared__ double red_v[PANEL_THREADS / 32];
  __shared__ int red_i[PANEL_THREADS / 32];

  const int cs = (int)cluster_nctarank();
  const int rank = (int)cluster_ctarank();
  const int item = blockIdx.x / cs;
  const int n = p.a.n, ld = p.a.ld, nb = p.nb, j0 = p.j0, rhp = p.rhp;
  double* X = p.a.base + (long long)p.slots[item] * p.a.slot_elems;
  int* orig = reinterpret_cast<int*>(psm + (long long)nb * rhp);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int row_lo = j0 + rank * p.rh;
  int myrows = n - row_lo;
  myrows = myrows < 0 ? 0 : (myrows > p.rh ? p.rh : myrows);

  // load my slab of the panel (X-columns j0..j0+nb-1 are contiguous memory rows)
  for (int c = 0; c < nb; ++c)
    for (int i = tid; i < myrows; i += PANEL_THREADS)
      psm[c * rhp + i] = X[(row_lo + i) + (long long)(j0 + c) * ld];
  for (int i = tid; i < myrows; i += PANEL_THREADS) orig[i] = row_lo + i;
  if (cs > 1) cluster_sync_all(); else __syncthreads();

  for (int jj = 0; jj < nb; ++jj) {
    const int j = j0 + jj;
    const int par = jj & 1;
    // (a) CTA-local argmax of |x| over rows >= j
    double bv = -1.0;
    int bi = INT_MAX;
    for (int i = tid; i < myrows; i += PANEL_THREADS) {
      const int gi = row_lo + i;
      if (gi >= j) argmax_merge(bv, bi, fabs(psm[jj * rhp + i]), gi);
    }
    warp_argmax(bv, bi);
    if (lane == 0) {
      red_v[warp] = bv;
      red_i[warp] = bi;
    }
    __syncthreads();
    if (warp == 0) {
      bv = lane < PANEL_THREADS / 32 ? red_v[lane] : -1.0;
      bi = lane < PANEL_THREADS / 32 ? red_i[lane] : INT_MAX;
      warp_argmax(bv, bi);
      const int li = bi - row_lo;
      const bool have = bi != INT_MAX;
      for (int d = 0; d < cs; ++d) {
        if (lane == 0) {
          dsmem_st_f64(dsmem_addr(&cand_val[par][rank], d), bv);
          dsmem_st_s32(dsmem_addr(&cand_idx[par][rank], d), bi);
          dsmem_st_s32(dsmem_addr(&cand_orig[par][rank], d), have ? orig[li] : -1);
        }
        if (have && lane < nb)
          dsmem_st_f64(dsmem_addr(&cand_row[par][rank][lane], d), psm[lane * rhp + li]);
      }
    }
    // (b) the owner of row j publishes it (it is what the pivot row swaps with)
    if (warp == 1 && j >= row_lo && j < row_lo + myrows) {
      const int lj = j - row_lo;
      for (int d = 0; d < cs; ++d) {
        if (lane < nb) dsmem_st_f64(dsmem_addr(&rowj[par][lane], d), psm[lane * rhp + lj]);
        if (lane == 0) dsmem_st_s32(dsmem_addr(&rowj_orig[par], d), orig[lj]);
      }
    }
    if (cs > 1) cluster_sync_all(); else __syncthreads();

    // (c) cluster-wide winner (identical in every CTA)
    double wv = -1.0;
    int wi = INT_MAX, wr = 0;
    for (int d = 0; d < cs; ++d) {
      const double v = cand_val[par][d];
      const int ix = cand_idx[par][d];
      if (v > wv || (v == wv && ix < wi)) {
        wv = v;
        wi = ix;
        wr = d;
      }
    }
    const bool none = (wi == INT_MAX);  // all NaN: idamax returns the first index
    const int pr = none ? j : wi;
    const double* urow = none ? rowj[par] : cand_row[par][wr];
    const int uorig = none ? rowj_orig[par] : cand_orig[par][wr];
    const double piv = urow[jj];
    if (tid == 0 && rank == 0) p.ipiv[(long long)item * p.n_stride + j] = pr;
    // (d) interchange rows j and pr (dgetf2 swaps only for a nonzero pivot)
    if (pr != j && piv != 0.0) {
      if (j >= row_lo && j < row_lo + myrows) {
        const int lj = j - row_lo;
        if (tid < nb) psm[tid * rhp + lj] = urow[tid];
        if (tid == 0) orig[lj] = uorig;
      }
      if (pr >= row_lo && pr < row_lo + myrows) {
        const int lp = pr - row_lo;
        if (tid < nb) psm[tid * rhp + lp] = rowj[par][tid];
        if (tid == 0) orig[lp] = rowj_orig[par];
      }
    }
    __syncthreads();
    // (e) scale the column below the pivot and rank-1 update the panel; the
    // pivot row is hoisted into registers so the per-row updates are
    // independent smem read-modify-writes (no aliasing chains)
    double u[NBMAX];
#pragma unroll
    for (int c = 0; c < NBMAX; ++c) u[c] = (c > jj && c < nb) ? urow[c] : 0.0;
    const bool recip = fabs(piv) >= kSfmin;
    const double rinv = 1.0 / piv;
    for (int i = tid; i < myrows; i += PANEL_THREADS) {
      const int gi = row_lo + i;
      if (gi <= j) continue;
      double l = psm[jj * rhp + i];
      if (piv != 0.0) l = recip ? l * rinv : l / piv;
      psm[jj * rhp + i] = l;
#pragma unroll
      for (int c = 0; c < NBMAX; ++c)
        if (c > jj && c < nb) psm[c * rhp + i] = fma(-l, u[c], psm[c * rhp + i]);
    }
    __syncthreads();
  }

  // write back; publish the interchange map for the rowpanel kernel
  for (int c = 0; c < nb; ++c)
    for (int i = tid; i < myrows; i += PANEL_THREADS)
      X[(row_lo + i) + (long long)(j0 + c) * ld] = psm[c * rhp + i];
  int* sig = p.sigma + (long long)item * p.n_stride;
  int* pairs = p.pairs + (long long)item * p.pair_stride + (long long)p.pidx * (1 + 2 * NBMAX);
  for (int i = tid; i < myrows; i += PANEL_THREADS) {
    const int gi = row_lo + i;
    const int o = orig[i];
    if (gi < j0 + nb) {
      sig[gi] = o;
    } else if (o != gi) {
      const int q = atomicAdd(pairs, 1);
      pairs[1 + 2 * q] = gi;
      pairs[2 + 2 * q] = o;
    }
  }
  // no CTA may exit while a peer could still address its shared memory
  if (cs > 1) cluster_sync_all();
}

// --------------------------------------------------------------- rowpanel
struct RowPanelArgs {
  ArenaView a;
  const int* slots;
  int j0, nb, pidx;
  const int* sigma;
  const int* pairs;
  int* pi;
  int n_stride, pair_stride;
};

constexpr int RP_THREADS = 128;

__global__ void __launch_bounds__(RP_THREADS) rowpanel_kernel(RowPanelArgs p) {
  __shared__ double L[NBMAX][NBMAX + 1];
  __shared__ int sig[NBMAX];
  __shared__ int prs[1 + 2 * NBMAX];
  const int item = blockIdx.y;
  const int n = p.a.n, ld = p.a.ld, nb = p.nb, j0 = p.j0;
  double* X = p.a.base + (long long)p.slots[item] * p.a.slot_elems;
  const int* pairs = p.pairs + (long long)item * p.pair_stride + (long long)p.pidx * (1 + 2 * NBMAX);
  const int tid = threadIdx.x;
  if (tid < nb) sig[tid] = p.sigma[(long long)item * p.n_stride + j0 + tid];
  if (tid == 0) prs[0] = pairs[0];
  __syncthreads();
  const int cnt = prs[0];
  for (int q = tid; q < 2 * cnt; q += RP_THREADS) prs[1 + q] = pairs[1 + q];

  if (blockIdx.x == gridDim.x - 1) {
    // compose the panel's interchanges into the running row permutation pi
    int* pi = p.pi + (long long)item * p.n_stride;
    __syncthreads();
    int va = 0, vb = 0;
    if (tid < nb) va = pi[sig[tid]];
    if (tid < cnt) vb = pi[prs[2 + 2 * tid]];
    __syncthreads();
    if (tid < nb) pi[j0 + tid] = va;
    if (tid < cnt) pi[prs[1 + 2 * tid]] = vb;
    return;
  }

  for (int e = tid; e < nb * nb; e += RP_THREADS) {
    const int i = e % nb, c = e / nb;
    L[i][c] = X[(j0 + i) + (long long)(j0 + c) * ld];
  }
  __syncthreads();

  const int c = blockIdx.x * RP_THREADS + tid;
  const int cc = c < j0 ? c : c + nb;  // skip the panel's own columns
  if (cc >= n) return;
  double* col = X + (long long)cc * ld;
  double seg[NBMAX];
  double ov[NBMAX];
#pragma unroll
  for (int i = 0; i < NBMAX; ++i)
    if (i < nb) seg[i] = col[sig[i]];
#pragma unroll
  for (int q = 0; q < NBMAX; ++q)
    if (q < cnt) ov[q] = col[prs[2 + 2 * q]];
#pragma unroll
  for (int q = 0; q < NBMAX; ++q)
    if (q < cnt) col[prs[1 + 2 * q]] = ov[q];
  if (cc >= j0 + nb) {
    // U12 = L11^-1 A12 (dtrsm Left/Lower/NoTrans/Unit order)
#pragma unroll
    for (int k = 0; k < NBMAX; ++k) {
      if (k < nb) {
        const double xk = seg[k];
#pragma unroll
        for (int i = k + 1; i < NBMAX; ++i)
          if (i < nb) seg[i] = fma(-xk, L[i][k], seg[i]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NBMAX; ++i)
    if (i < nb) col[j0 + i] = seg[i];
}

// ------------------------------------------------------------- diag check
__global__ void diag_check_kernel(ArenaView a, const int* slots, const unsigned long long* scale_bits,
                                  int* status) {
  __shared__ int first;
  const int item = blockIdx.x;
  const double* X = a.base + (long long)slots[item] * a.slot_elems;
  const double scale = __longlong_as_double((long long)scale_bits[item]);
  const double tol = (double)a.n * kEps * scale;
  if (threadIdx.x == 0) first = INT_MAX;
  __syncthreads();
  for (int i = threadIdx.x; i < a.n; i += blockDim.x) {
    const double d = fabs(X[i + (long long)i * a.ld]);
    if (!(d > tol)) atomicMin(&first, i);
  }
  __syncthreads();
  if (threadIdx.x == 0) status[item] = first == INT_MAX ? 0 : first + 1;
}

}  // namespace

// ======================================================================
cudaError_t launch_maxabs(const ArenaView& a, const int* slots, int count,
                          unsigned long long* scale_bits, cudaStream_t s) {
  const long long total = (long long)a.n * a.n;
  int blocks = (int)((total + 255) / 256);
  blocks = blocks > 64 ? 64 : (blocks < 1 ? 1 : blocks);
  count_launch();
  maxabs_kernel<<<dim3(blocks, count), 256, 0, s>>>(a, slots, scale_bits);
  return cudaGetLastError();
}

cudaError_t launch_copy(const ArenaView& a, const int* pairs, int count, cudaStream_t s) {
  const int gx = a.n < 512 ? a.n : 512;
  count_launch();
  copy_kernel<<<dim3(gx, count), 256, 0, s>>>(a, pairs);
  return cudaGetLastError();
}

cudaError_t launch_permcopy(const ArenaView& a, const int* pairs, int count, const int* pi,
                            int pi_stride, bool identity_src, cudaStream_t s) {
  const int gx = a.n < 512 ? a.n : 512;
  count_launch();
  permcopy_kernel<<<dim3(gx, count), 256, 0, s>>>(a, pairs, pi, pi_stride, identity_src ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_pi_init(int* pi, int n, int count, cudaStream_t s) {
  count_launch();
  pi_init_kernel<<<dim3((n + 255) / 256, count), 256, 0, s>>>(pi, n);
  return cudaGetLastError();
}

int panel_width(int n) {
  // widest panel whose full height fits the distributed smem of an 8-CTA cluster
  int nb = NBMAX;
  while (nb > 8 && (long long)n * nb * 8 > (long long)MAXCS * 180 * 1024) nb >>= 1;
  return nb;
}

static int panel_cluster_size(int h, int nb) {
  // keep a CTA's slab of the panel under ~150 KB of shared memory
  const long long bytes = (long long)h * nb * 8;
  int cs = 1;
  while (cs < MAXCS && bytes > (long long)cs * 150 * 1024) cs *= 2;
  return cs;
}

cudaError_t launch_panel(const ArenaView& a, const int* slots, int count, int j0, int nb, int pidx,
                         const LuScratch& sc, int n_stride, int pair_stride, cudaStream_t s) {
  const int h = a.n - j0;
  const int cs = panel_cluster_size(h, nb);
  PanelArgs p;
  p.a = a;
  p.slots = slots;
  p.j0 = j0;
  p.nb = nb;
  p.pidx = pidx;
  p.rh = (h + cs - 1) / cs;
  p.rhp = (p.rh + 1) | 1;  // odd stride: spreads column accesses over banks
  p.ipiv = sc.ipiv;
  p.sigma = sc.sigma;
  p.pairs = sc.pairs;
  p.n_stride = n_stride;
  p.pair_stride = pair_stride;
  const size_t smem = (size_t)nb * p.rhp * 8 + (size_t)p.rhp * 4 + 16;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(lu_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         200 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(count * cs);
  cfg.blockDim = dim3(PANEL_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  count_launch();
  return cudaLaunchKernelEx(&cfg, lu_panel_kernel, p);
}

cudaError_t launch_rowpanel(const ArenaView& a, const int* slots, int count, int j0, int nb, int pidx,
                            const LuScratch& sc, int n_stride, int pair_stride, cudaStream_t s) {
  RowPanelArgs p;
  p.a = a;
  p.slots = slots;
  p.j0 = j0;
  p.nb = nb;
  p.pidx = pidx;
  p.sigma = sc.sigma;
  p.pairs = sc.pairs;
  p.pi = sc.pi;
  p.n_stride = n_stride;
  p.pair_stride = pair_stride;
  const int cols = a.n - nb;
  const int gx = (cols + RP_THREADS - 1) / RP_THREADS + 1;  // +1: the pi-update block
  count_launch();
  rowpanel_kernel<<<dim3(gx, count), RP_THREADS, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_diag_check(const ArenaView& a, const int* slots, int count,
                              const unsigned long long* scale_bits, int* status, cudaStream_t s) {
  count_launch();
  diag_check_kernel<<<count, 256, 0, s>>>(a, slots, scale_bits, status);
  return cudaGetLastError();
}

}  // namespace bri
