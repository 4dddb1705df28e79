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

constexpr int PORTABLE_CS = 8;      // preferred cluster size cap (portable)
constexpr int MAXCS = 16;           // non-portable clusters for panels taller than 8 x 2 x PT rows

// ----------------------------------------------------------------- maxabs
// max |X| per slot (the scale of the singularity test, core.py:200-209).  One
// CTA row per X-column group, coalesced along the contiguous dimension; the
// bit-pattern max lets NaN (positive, above +Inf) propagate like numpy's max.
__global__ void maxabs_kernel(ArenaView a, const int* slots, unsigned long long* out) {
  const int item = blockIdx.y;
  const double* x = a.base + (long long)slots[item] * a.slot_elems;
  long long best = 0;
  for (int j = blockIdx.x; j < a.n; j += gridDim.x) {
    const double* col = x + (long long)j * a.ld;
    for (int i = threadIdx.x; i < a.n; i += blockDim.x) {
      const long long v = __double_as_longlong(fabs(col[i]));
      best = v > best ? v : best;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const long long o = __shfl_xor_sync(0xffffffffu, best, off);
    best = o > best ? o : best;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out + item, (unsigned long long)best);
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

// X-column x of src -> X-column pi[x] of dst (memory rows, coalesced)
__global__ void colscatter_kernel(ArenaView a, const int* pairs, const int* pi, int pi_stride) {
  const int item = blockIdx.y;
  const double* src = a.base + (long long)pairs[2 * item] * a.slot_elems;
  double* dst = a.base + (long long)pairs[2 * item + 1] * a.slot_elems;
  const int* p = pi + (long long)item * pi_stride;
  for (int x = blockIdx.x; x < a.n; x += gridDim.x) {
    const double* s = src + (long long)x * a.ld;
    double* d = dst + (long long)p[x] * a.ld;
    for (int i = threadIdx.x; i < a.n; i += blockDim.x) d[i] = s[i];
  }
}

__global__ void identity_kernel(ArenaView a, const int* slots, int slot_stride) {
  double* x = a.base + (long long)slots[slot_stride * blockIdx.y] * a.slot_elems;
  for (int j = blockIdx.x; j < a.n; j += gridDim.x)
    for (int i = threadIdx.x; i < a.n; i += blockDim.x) x[i + (long long)j * a.ld] = (i == j) ? 1.0 : 0.0;
}

__global__ void pi_init_kernel(int* pi, int n) {
  const int item = blockIdx.y;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x)
    pi[(long long)item * n + x] = x;
}

// ------------------------------------------------------------------ panel
// The (n - j0) x nb panel (nb <= 32) is spread over a cluster of cs CTAs of
// PT threads; thread t of CTA r owns rows row_lo + q*PT + t (q < RPT) and keeps
// their not-yet-final values in registers, *shifted*: after column jj,
// x[q][c] holds column jj+1+c.  The shift keeps every register index static
// while the column loop stays rolled (a fully unrolled panel overflowed the
// instruction cache: 46% no_instruction stalls).  Finished values — the
// multipliers (L) of every row and the U rows of the pivots — live in shared
// memory psm[c * rhp + i] and are written back at the end.  Row buffers are
// 64 wide with a zero upper half, so shifted reads need no predicates.
// Per column jj (pivot position j = j0 + jj):
//   (1) thread candidate, warp shuffle argmax; each warp's winning lane
//       stores its row (L part from psm by the lanes, live part from its
//       registers) to wrow[warp]; the owner of row j stores row j -> barrier
//   (2) every thread picks the CTA winner from the PW slots
//   (3) cs > 1: warp 0 pushes the CTA candidate row to every CTA (DSMEM),
//       warp 1 of row j's owner pushes row j -> cluster barrier
//   (4) every thread picks the global winner; rows j and p are exchanged
//       (pivot row final in psm); active rows scale and rank-1 update (31 DFMA).
#ifdef BRI_PANEL_PROFILE
__device__ unsigned long long g_panel_phase[8];
#define PPROF(k)                                                         \
  do {                                                                   \
    if (threadIdx.x == 0 && blockIdx.x == 0) {                           \
      const unsigned long long now = clock64();                          \
      g_panel_phase[k] += now - t_last;                                  \
      t_last = now;                                                      \
    }                                                                    \
  } while (0)
#else
#define PPROF(k) do { } while (0)
#endif
constexpr int PT = 256;
constexpr int PW = PT / 32;
constexpr int PNB = NBMAX;      // live register width (narrower panels are zero-padded)
constexpr int RW = 2 * PNB;     // row buffer width (upper half zero)

struct PanelArgs {
  ArenaView a;
  const int* slots;
  int j0, nb, rows_per_cta, rhp, pidx;
  int* ipiv;
  int* sigma;
  int* pairs;
  int n_stride, pair_stride;
};


// The owning lane stores its live row, shifted (x[c] -> dst[c + 1]), with
// 16-byte stores; dst is a 16-byte aligned 34-wide buffer (tail stays zero).
template <int RPT>
BRI_DEVI void store_live_row(double* dst, const double (&x)[RPT][PNB], int q) {
  double r[PNB];
#pragma unroll
  for (int c = 0; c < PNB; ++c) {
    r[c] = x[0][c];
#pragma unroll
    for (int qq = 1; qq < RPT; ++qq)
      if (q == qq) r[c] = x[qq][c];
  }
  dst[1] = r[0];
#pragma unroll
  for (int c = 1; c < PNB - 1; c += 2) sts_f64x2(&dst[c + 1], r[c], r[c + 1]);
  dst[PNB] = r[PNB - 1];
}

template <int RPT>
__global__ void __launch_bounds__(PT, 1) lu_panel_kernel(PanelArgs p) {
  // Row buffers are split: L part (columns < jj) and the live part in
  // *shifted* coordinates, x[c] (column jj + c) stored at index c + 1 of a
  // 34-wide buffer whose tail is zero, so the update reads u[c] = buf[c + 2]
  // with aligned 16-byte loads.
  constexpr int SW = 34;
  // one 544-byte message per row: L part, shifted live part, (value, row, origin)
  struct __align__(16) RowMsg {
    double L[PNB];
    double S[SW];
    double val;
    int idx, orig;
  };
  static_assert(sizeof(RowMsg) % 16 == 0, "bulk copies move 16-byte multiples");
  extern __shared__ double psm[];                       // nb columns x rhp rows, then rhp ints
  __shared__ double wval[2][PW];
  __shared__ int widx[2][PW];
  __shared__ RowMsg cmsg[2][MAXCS];                     // candidates, by source CTA rank
  __shared__ RowMsg jmsg[2];                            // row j, from its owner CTA
  __shared__ RowMsg cstg[2], jstg[2];                   // local staging of outgoing messages (cs > 1)
  __shared__ __align__(8) uint64_t xbar[2];             // exchange mbarriers (cs > 1)

  const int cs = (int)cluster_nctarank();
  const int rank = (int)cluster_ctarank();
  const int item = blockIdx.x / cs;
  const int n = p.a.n, ld = p.a.ld, nb = p.nb, j0 = p.j0, rhp = p.rhp;
  double* X = p.a.base + (long long)p.slots[item] * p.a.slot_elems;
  int* orig = reinterpret_cast<int*>(psm + (long long)nb * rhp);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int row_lo = j0 + rank * p.rows_per_cta;
  const int myrows = max(0, min(n, row_lo + p.rows_per_cta) - row_lo);
  // bytes each CTA receives per column: cs candidates + row j
  const uint32_t xbytes = (uint32_t)(cs + 1) * (uint32_t)sizeof(RowMsg);

  for (int e = tid; e < 2 * MAXCS * SW; e += PT) cmsg[e / (MAXCS * SW)][(e / SW) % MAXCS].S[e % SW] = 0.0;
  for (int e = tid; e < 2 * SW; e += PT) {
    jmsg[e / SW].S[e % SW] = 0.0;
    cstg[e / SW].S[e % SW] = 0.0;
    jstg[e / SW].S[e % SW] = 0.0;
  }
  if (tid == 0) {
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    fence_barrier_init();
  }

  double x[RPT][PNB];
  int gi[RPT];
  bool valid[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int li = q * PT + tid;
    gi[q] = row_lo + li;
    valid[q] = li < myrows;
#pragma unroll
    for (int c = 0; c < PNB; ++c)
      x[q][c] = (valid[q] && c < nb) ? X[gi[q] + (long long)(j0 + c) * ld] : 0.0;
    if (valid[q]) orig[li] = gi[q];
  }
  // candidate for column 0
  double bv = -1.0;
  int bi = INT_MAX, bq = 0;
#pragma unroll
  for (int q = 0; q < RPT; ++q)
    if (valid[q]) {
      const double v = fabs(x[q][0]);
      if (v > bv || (v == bv && gi[q] < bi)) { bv = v; bi = gi[q]; bq = q; }
    }
  {
    double wv = bv;
    int wi = bi;
    warp_argmax_fast(wv, wi);
    if (lane == 0) { wval[0][warp] = wv; widx[0][warp] = wi; }
  }
  if (cs > 1) cluster_sync_all(); else __syncthreads();
#ifdef BRI_PANEL_PROFILE
  unsigned long long t_last = clock64();
#endif

  for (int jj = 0; jj < nb; ++jj) {
    const int j = j0 + jj;
    const int par = jj & 1;
    if (cs > 1 && tid == 0) mbar_arrive_expect_tx(&xbar[par], xbytes);
    // ---- (2) CTA winner from the warp slots (written at the end of the previous column)
    double cv = wval[par][lane % PW];
    int ci = widx[par][lane % PW];
    warp_argmax_fast(cv, ci);
    PPROF(0);
    // ---- (3) publish: the CTA winner's row and row j, by their owning warps
    const bool have = ci != INT_MAX;
    const int lw = ci - row_lo;                    // local index of the CTA winner
    const bool own_j = (j >= row_lo && j < row_lo + myrows);
    const int lj = j - row_lo;
    uint32_t aL, aS, bL, bS;
    int pr, uorig, jorig;
    if (cs > 1) {
      // stage our CTA candidate (and row j if we own it) as one message each,
      // then one lane bulk-copies it into slot `rank` of every CTA of the cluster
      if (have && warp == ((lw % PT) >> 5)) {
        if (lane == (lw & 31)) {
          store_live_row<RPT>(cstg[par].S, x, lw / PT);
          cstg[par].val = cv;
          cstg[par].idx = ci;
          cstg[par].orig = orig[lw];
        }
        cstg[par].L[lane] = lane < jj ? psm[lane * rhp + lw] : 0.0;
      } else if (!have && warp == 0) {
        cstg[par].L[lane] = 0.0;
        if (lane == 0) {
          cstg[par].val = -1.0;
          cstg[par].idx = INT_MAX;
          cstg[par].orig = -1;
        }
      }
      if (own_j && warp == ((lj % PT) >> 5)) {
        if (lane == (lj & 31)) {
          store_live_row<RPT>(jstg[par].S, x, lj / PT);
          jstg[par].orig = orig[lj];
        }
        jstg[par].L[lane] = lane < jj ? psm[lane * rhp + lj] : 0.0;
      }
      const bool pub_c = (have && warp == ((lw % PT) >> 5)) || (!have && warp == 0);
      const bool pub_j = own_j && warp == ((lj % PT) >> 5);
      if (pub_c || pub_j) {
        fence_proxy_async_smem();   // generic smem writes -> visible to the bulk-copy engine
        __syncwarp();
        // one destination per lane: the bulk copies are issued in parallel
        if (pub_c && lane < cs)
          bulk_s2cluster(dsmem_addr(&cmsg[par][rank], lane), &cstg[par], sizeof(RowMsg), dsmem_addr(&xbar[par], lane));
        if (pub_j && lane >= 16 && lane < 16 + cs)
          bulk_s2cluster(dsmem_addr(&jmsg[par], lane - 16), &jstg[par], sizeof(RowMsg),
                         dsmem_addr(&xbar[par], lane - 16));
      }
      PPROF(1);
      mbar_wait_cluster(&xbar[par], (jj >> 1) & 1);
      PPROF(2);
      double gv = lane < cs ? cmsg[par][lane].val : -1.0;
      int gidx = lane < cs ? cmsg[par][lane].idx : INT_MAX;
      const int myidx = gidx;
      warp_argmax_fast(gv, gidx);
      const int gr = __ffs(__ballot_sync(0xffffffffu, lane < cs && gidx != INT_MAX && myidx == gidx)) - 1;
      const bool none = gidx == INT_MAX;  // all NaN: idamax returns the first index
      pr = none ? j : gidx;
      aL = none ? smem_u32(jmsg[par].L) : smem_u32(cmsg[par][gr].L);
      aS = none ? smem_u32(jmsg[par].S) : smem_u32(cmsg[par][gr].S);
      uorig = none ? jmsg[par].orig : cmsg[par][gr].orig;
      jorig = jmsg[par].orig;
    } else {
      if (have && warp == ((lw % PT) >> 5)) {
        if (lane == (lw & 31)) {
          store_live_row<RPT>(cmsg[par][0].S, x, lw / PT);
          cmsg[par][0].orig = orig[lw];
        }
        if (lane < jj) cmsg[par][0].L[lane] = psm[lane * rhp + lw];
      }
      if (own_j && warp == ((lj % PT) >> 5)) {
        if (lane == (lj & 31)) {
          store_live_row<RPT>(jmsg[par].S, x, lj / PT);
          jmsg[par].orig = orig[lj];
        }
        if (lane < jj) jmsg[par].L[lane] = psm[lane * rhp + lj];
      }
      PPROF(1);
      __syncthreads();
      PPROF(2);
      pr = have ? ci : j;
      aL = have ? smem_u32(cmsg[par][0].L) : smem_u32(jmsg[par].L);
      aS = have ? smem_u32(cmsg[par][0].S) : smem_u32(jmsg[par].S);
      uorig = have ? cmsg[par][0].orig : jmsg[par].orig;
      jorig = jmsg[par].orig;
    }
    bL = smem_u32(jmsg[par].L);
    bS = smem_u32(jmsg[par].S);
    PPROF(3);
    // ---- (4) interchange, scale, rank-1 update; the next column's candidate
    //          is formed as soon as its values are updated
    const double piv = lds_f64(aS + 8);
    if (tid == 0 && rank == 0) p.ipiv[(long long)item * p.n_stride + j] = pr;
    const bool swap = (pr != j && piv != 0.0);  // dgetf2 interchanges only for a nonzero pivot
    const bool recip = fabs(piv) >= kSfmin;
    const double rinv = 1.0 / piv;
    if (own_j && warp == ((lj % PT) >> 5)) {    // position j: the pivot row, final
      const uint32_t sL = swap ? aL : bL, sS = swap ? aS : bS;
      if (lane < nb) psm[lane * rhp + lj] = lane < jj ? lds_f64(sL + 8 * lane) : lds_f64(sS + 8 * (lane - jj + 1));
      if (lane == 0 && swap) orig[lj] = uorig;
    }
    const bool own_p = swap && pr >= row_lo && pr < row_lo + myrows;
    const int lp = pr - row_lo;
    if (own_p && warp == ((lp % PT) >> 5)) {    // position p: old row j's L part
      if (lane < jj) psm[lane * rhp + lp] = lds_f64(bL + 8 * lane);
      if (lane == 0) orig[lp] = jorig;
    }
    PPROF(4);
    double u[PNB];
#pragma unroll
    for (int c = 0; c < PNB; c += 2) lds_f64x2(aS + 16 + 8 * c, u[c], u[c + 1]);
    double nl[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      nl[q] = 0.0;
      if (!valid[q] || gi[q] <= j) continue;
      if (own_p && gi[q] == pr) {
#pragma unroll
        for (int c = 0; c < PNB; ++c) x[q][c] = lds_f64(bS + 8 * (c + 1));
      }
      double l = x[q][0];
      if (piv != 0.0) l = recip ? l * rinv : l / piv;
      nl[q] = l;
      psm[jj * rhp + q * PT + tid] = l;
      x[q][0] = fma(-l, u[0], x[q][1]);  // next column first
    }
    // next column's candidate + warp reduction (overlaps the remaining updates)
    bv = -1.0;
    bi = INT_MAX;
#pragma unroll
    for (int q = 0; q < RPT; ++q)
      if (valid[q] && gi[q] > j) {
        const double v = fabs(x[q][0]);
        if (v > bv || (v == bv && gi[q] < bi)) { bv = v; bi = gi[q]; bq = q; }
      }
    {
      double wv = bv;
      int wi = bi;
      warp_argmax_fast(wv, wi);
      if (lane == 0) { wval[par ^ 1][warp] = wv; widx[par ^ 1][warp] = wi; }
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      if (!valid[q] || gi[q] <= j) continue;
#pragma unroll
      for (int c = 1; c < PNB - 1; ++c) x[q][c] = fma(-nl[q], u[c], x[q][c + 1]);
      x[q][PNB - 1] = 0.0;
    }
    PPROF(5);
    __syncthreads();   // warp slots of the next column complete; rows j/p settled
  }

  // write back; publish the interchange map for the rowpanel kernel
  for (int e = tid; e < nb * myrows; e += PT) {
    const int c = e / myrows, i = e % myrows;
    X[(row_lo + i) + (long long)(j0 + c) * ld] = psm[c * rhp + i];
  }
  int* sig = p.sigma + (long long)item * p.n_stride;
  int* pairs = p.pairs + (long long)item * p.pair_stride + (long long)p.pidx * (1 + 2 * NBMAX);
  for (int i = tid; i < myrows; i += PT) {
    const int g = row_lo + i, o = orig[i];
    if (g < j0 + nb) {
      sig[g] = o;
    } else if (o != g) {
      const int k = atomicAdd(pairs, 1);
      pairs[1 + 2 * k] = g;
      pairs[2 + 2 * k] = o;
    }
  }
  // no CTA may exit while a peer could still address its shared memory
  if (cs > 1) cluster_sync_all();
}

// --------------------------------------------------------------- rowpanel
// One warp per X-column outside the panel (a contiguous memory row): apply
// the panel's interchanges as a gather (all reads before any write, ordered
// by __syncwarp) and, right of the panel, solve L11 * U12 = A12 across the
// lanes (lane i owns row j0 + i; forward substitution with shuffles).
struct RowPanelArgs {
  ArenaView a;
  const int* slots;
  int j0, nb, pidx;
  int cbeg, cend;     // X-columns handled: [cbeg, cend) minus the panel's own
  const int* sigma;
  const int* pairs;
  int* pi;
  int n_stride, pair_stride;
};

constexpr int RP_THREADS = 256;

__global__ void __launch_bounds__(RP_THREADS) rowpanel_kernel(RowPanelArgs p) {
  __shared__ double L[NBMAX][NBMAX + 1];
  __shared__ int sig[NBMAX];
  __shared__ int prs[1 + 2 * NBMAX];
  const int item = blockIdx.y;
  const int n = p.a.n, ld = p.a.ld, nb = p.nb, j0 = p.j0;
  double* X = p.a.base + (long long)p.slots[item] * p.a.slot_elems;
  const int* pairs = p.pairs + (long long)item * p.pair_stride + (long long)p.pidx * (1 + 2 * NBMAX);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
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

  const int c = p.cbeg + blockIdx.x * (RP_THREADS / 32) + warp;
  const bool inside = (j0 >= p.cbeg && j0 < p.cend);
  const int cc = (inside && c >= j0) ? c + nb : c;  // skip the panel's own columns
  if (cc >= p.cend || cc >= n) return;
  double* col = X + (long long)cc * ld;
  const double seg = lane < nb ? col[sig[lane]] : 0.0;
  const double ov = lane < cnt ? col[prs[2 + 2 * lane]] : 0.0;
  __syncwarp();
  if (lane < cnt) col[prs[1 + 2 * lane]] = ov;
  double xv = seg;
  if (cc >= j0 + nb) {
    // U12 = L11^-1 A12 (dtrsm Left/Lower/NoTrans/Unit order)
    for (int k = 0; k < nb - 1; ++k) {
      const double xk = __shfl_sync(0xffffffffu, xv, k);
      if (lane > k && lane < nb) xv = fma(-xk, L[lane][k], xv);
    }
  }
  if (lane < nb) col[j0 + lane] = xv;
}

// ---------------------------------------------------------------- laswp
// Apply the interchanges of npan consecutive inner panels (starting at panel
// index pidx0, rows j0q = J0 + q * nbi) to X-columns [0, J0) and [J0 + W, n):
// one warp per column, each panel as a gather (reads, __syncwarp, writes).
struct LaswpArgs {
  ArenaView a;
  const int* slots;
  int J0, W, nbi, pidx0, npan;
  int a0, a1, b0, b1;   // X-columns handled: [a0, a1) then [b0, b1)
  const int* sigma;
  const int* pairs;
  int n_stride, pair_stride;
};

__global__ void __launch_bounds__(RP_THREADS) laswp_kernel(LaswpArgs p) {
  const int item = blockIdx.y;
  const int n = p.a.n, ld = p.a.ld;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * (RP_THREADS / 32) + warp;
  const int na = p.a1 - p.a0;
  const int cc = c < na ? p.a0 + c : p.b0 + (c - na);
  if (c >= na && cc >= p.b1) return;
  double* col = p.a.base + (long long)p.slots[item] * p.a.slot_elems + (long long)cc * ld;
  const int* sig = p.sigma + (long long)item * p.n_stride;
  for (int q = 0; q < p.npan; ++q) {
    const int j0 = p.J0 + q * p.nbi;
    const int w = min(p.nbi, n - j0);
    const int* pr = p.pairs + (long long)item * p.pair_stride + (long long)(p.pidx0 + q) * (1 + 2 * NBMAX);
    const int cnt = pr[0];
    const double seg = lane < w ? col[sig[j0 + lane]] : 0.0;
    const double ov = lane < cnt ? col[pr[2 + 2 * lane]] : 0.0;
    __syncwarp();
    if (lane < cnt) col[pr[1 + 2 * lane]] = ov;
    if (lane < w) col[j0 + lane] = seg;
    __syncwarp();
  }
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

#ifdef BRI_PANEL_PROFILE
void panel_profile_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_panel_phase, sizeof(g_panel_phase));
  unsigned long long z[8] = {0};
  cudaMemcpyToSymbol(g_panel_phase, z, sizeof(z));
}
#endif

// ======================================================================
cudaError_t launch_maxabs(const ArenaView& a, const int* slots, int count,
                          unsigned long long* scale_bits, cudaStream_t s) {
  int blocks = a.n < 1024 ? a.n : 1024;
  if (count > 16) blocks = (blocks + 15) / 16;
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

cudaError_t launch_colscatter(const ArenaView& a, const int* pairs, int count, const int* pi, int pi_stride,
                              cudaStream_t s) {
  const int gx = a.n < 1024 ? a.n : 1024;
  count_launch();
  colscatter_kernel<<<dim3(gx, count), 256, 0, s>>>(a, pairs, pi, pi_stride);
  return cudaGetLastError();
}

cudaError_t launch_identity(const ArenaView& a, const int* slots, int slot_stride, int count, cudaStream_t s) {
  const int gx = a.n < 1024 ? a.n : 1024;
  count_launch();
  identity_kernel<<<dim3(gx, count), 256, 0, s>>>(a, slots, slot_stride);
  return cudaGetLastError();
}

cudaError_t launch_pi_init(int* pi, int n, int count, cudaStream_t s) {
  count_launch();
  pi_init_kernel<<<dim3((n + 255) / 256, count), 256, 0, s>>>(pi, n);
  return cudaGetLastError();
}

// Panel width: 32 columns, held in registers (up to 2 rows x 32 per thread).
int panel_width(int n) { return n > 0 ? NBMAX : NBMAX; }

template <int RPT>
static cudaError_t launch_panel_t(PanelArgs p, int cs, int count, cudaStream_t s) {
  const size_t smem = (size_t)p.nb * p.rhp * 8 + (size_t)p.rhp * 4 + 16;
  if (smem > 160 * 1024) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(count * cs);
  cfg.blockDim = dim3(PT);
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
  return cudaLaunchKernelEx(&cfg, lu_panel_kernel<RPT>, p);
}

cudaError_t configure_lu() {
  cudaError_t e = cudaFuncSetAttribute(lu_panel_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(lu_panel_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(lu_panel_kernel<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return e;
}

int max_panel_rows() { return MAXCS * 2 * PT; }

cudaError_t launch_panel(const ArenaView& a, const int* slots, int count, int j0, int nb, int pidx,
                         const LuScratch& sc, int n_stride, int pair_stride, cudaStream_t s) {
  const int h = a.n - j0;
  // 1 row per thread while it fits a cluster of 8, else 2 (registers: 2 x 32 doubles)
  // Up to 8 x PT rows: 1 row per thread, portable clusters (measured: beats a
  // halved cluster at 2 rows); up to 8 x 2 x PT: 2 rows; beyond, 16-CTA clusters.
  const int rpt = h <= PORTABLE_CS * PT ? 1 : 2;
  int cs = 1;
  while (cs < MAXCS && (h + cs - 1) / cs > rpt * PT) cs <<= 1;
  if ((h + cs - 1) / cs > rpt * PT) return cudaErrorInvalidValue;  // order > max_panel_rows()
  PanelArgs p;
  p.a = a;
  p.slots = slots;
  p.j0 = j0;
  p.nb = nb;
  p.rows_per_cta = (h + cs - 1) / cs;
  p.rhp = p.rows_per_cta | 1;
  p.pidx = pidx;
  p.ipiv = sc.ipiv;
  p.sigma = sc.sigma;
  p.pairs = sc.pairs;
  p.n_stride = n_stride;
  p.pair_stride = pair_stride;
  if (rpt == 1) return launch_panel_t<1>(p, cs, count, s);
  return launch_panel_t<2>(p, cs, count, s);
}

cudaError_t launch_rowpanel(const ArenaView& a, const int* slots, int count, int j0, int nb, int pidx,
                            int cbeg, int cend, const LuScratch& sc, int n_stride, int pair_stride,
                            cudaStream_t s) {
  RowPanelArgs p;
  p.a = a;
  p.slots = slots;
  p.j0 = j0;
  p.nb = nb;
  p.pidx = pidx;
  p.cbeg = cbeg;
  p.cend = cend;
  p.sigma = sc.sigma;
  p.pairs = sc.pairs;
  p.pi = sc.pi;
  p.n_stride = n_stride;
  p.pair_stride = pair_stride;
  const int cols = (cend - cbeg) - ((j0 >= cbeg && j0 < cend) ? nb : 0);
  const int wpb = RP_THREADS / 32;
  const int gx = (cols + wpb - 1) / wpb + 1;  // +1: the pi-update block
  count_launch();
  rowpanel_kernel<<<dim3(gx, count), RP_THREADS, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_laswp(const ArenaView& a, const int* slots, int count, int J0, int W, int nbi, int pidx0,
                        int npan, int a0, int a1, int b0, int b1, const LuScratch& sc, int n_stride,
                        int pair_stride, cudaStream_t s) {
  a1 = a1 > a0 ? a1 : a0;
  b1 = b1 > b0 ? b1 : b0;
  const int cols = (a1 - a0) + (b1 - b0);
  if (cols <= 0) return cudaSuccess;
  LaswpArgs p;
  p.a0 = a0;
  p.a1 = a1;
  p.b0 = b0;
  p.b1 = b1;
  p.a = a;
  p.slots = slots;
  p.J0 = J0;
  p.W = W;
  p.nbi = nbi;
  p.pidx0 = pidx0;
  p.npan = npan;
  p.sigma = sc.sigma;
  p.pairs = sc.pairs;
  p.n_stride = n_stride;
  p.pair_stride = pair_stride;
  const int wpb = RP_THREADS / 32;
  count_launch();
  laswp_kernel<<<dim3((cols + wpb - 1) / wpb, count), RP_THREADS, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_diag_check(const ArenaView& a, const int* slots, int count,
                              const unsigned long long* scale_bits, int* status, cudaStream_t s) {
  count_launch();
  diag_check_kernel<<<count, 256, 0, s>>>(a, slots, scale_bits, status);
  return cudaGetLastError();
}

}  // namespace bri
