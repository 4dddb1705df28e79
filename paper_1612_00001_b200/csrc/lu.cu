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

#include <cstdlib>

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
                                int identity_src, const int* pidx) {
  const int item = blockIdx.y;
  const double* src = a.base + (long long)pairs[2 * item] * a.slot_elems;
  double* dst = a.base + (long long)pairs[2 * item + 1] * a.slot_elems;
  // pidx (optional): item -> factor index whose permutation applies (shared factors)
  const int* p = pi + (long long)(pidx ? pidx[item] : item) * pi_stride;
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

// Per-factorization scratch reset: pi = identity, the panels' interchange lists
// and the max|A| word zeroed (one kernel node instead of two graph memset nodes,
// which the CUPTI timeline showed waiting ~0.5 ms behind the preceding kernel).
__global__ void pi_init_kernel(int* pi, int n, unsigned long long* scale_bits, int* pairs, int pair_stride) {
  const int item = blockIdx.y;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  for (int x = tid; x < n; x += nth) pi[(long long)item * n + x] = x;
  for (int x = tid; x < pair_stride; x += nth) pairs[(long long)item * pair_stride + x] = 0;
  if (tid == 0) scale_bits[item] = 0ULL;
}

// ------------------------------------------------------------------ panel
// The (n - j0) x nb panel (nb <= 32) is spread over a cluster of cs CTAs of
// PT threads.  Thread t of CTA r owns the *slots* row_lo + q*PT + t (q < RPT):
// a slot is one original row of the panel, and its data never moves.  The
// not-yet-final values live in registers, *shifted*: after column jj, x[q][c]
// holds column jj+1+c (static register indices while the column loop stays
// rolled — a fully unrolled panel overflowed the instruction cache).  Each
// slot carries its current row position pos[q]; an interchange of rows j and
// p just exchanges two positions ("lazy relocation"), so no row ever travels
// between CTAs and the only data a column exchanges is the pivot candidates.
// Finished values — the multipliers (L) of every slot and the U rows of the
// pivots — live in shared memory psm[c * rhp + slot]; at the end every slot
// is written to its final position.
// Per column jj (pivot position j = j0 + jj):
//   (1) the CTA winner (largest |x|, smallest position on ties; NaNs never
//       win) from the per-warp slots written at the end of the previous column
//   (2) its owning thread stages the live row + (value, position) as one
//       288-byte message; cs > 1: the message is bulk-copied into slot `rank`
//       of every CTA of the cluster, completing on their exchange mbarrier
//   (3) every thread picks the global winner p from the cs candidates: the
//       pivot row (u) is read straight from the winning message
//   (4) positions j and p are exchanged (the finished pivot stores its U row),
//       active slots scale, form the next column first, reduce the next
//       candidate, then finish the rank-1 update (31 DFMA per slot).
// Pivot decisions are dgetf2's: idamax (first index on ties), interchange
// only for a nonzero pivot, reciprocal scaling when |pivot| >= sfmin; a
// column without any comparable value (all NaN) pivots in place.
#ifdef BRI_PANEL_PROFILE
__device__ unsigned long long g_panel_phase[10];
#define PPROF(k)                                                         \
  do {                                                                   \
    if (threadIdx.x == 0 && blockIdx.x == 0) {                           \
      const unsigned long long now = clock64();                          \
      ph_acc[k] += now - t_last;                                         \
      t_last = now;                                                      \
    }                                                                    \
  } while (0)
#else
#define PPROF(k) do { } while (0)
#endif
constexpr int PT = 256;
constexpr int PW = PT / 32;
constexpr int PNB = NBMAX;      // live register width (narrower panels are zero-padded)

struct PanelArgs {
  ArenaView a;
  const int* slots;
  int j0, nb, rows_per_cta, rhp, pidx;
  int* ipiv;
  int* sigma;
  int* pairs;
  int n_stride, pair_stride;
  int early;   // pdl_trigger before the wait (bri_internal.h)
};

// Live row of slot q, shifted (x[c] -> dst[c + 1]), with 16-byte stores; dst
// is a 16-byte aligned 34-wide buffer whose ends stay zero.
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
  for (int c = 1; c < PNB - 1; c += 2) *reinterpret_cast<double2*>(&dst[c + 1]) = make_double2(r[c], r[c + 1]);
  dst[PNB] = r[PNB - 1];
}

// The U row of a slot that just became pivot j0 + jj: its live values are
// columns jj.. of the panel.
BRI_DEVI void store_u_row(double* psm, int rhp, int jj, int nb, int slot, const double (&xr)[PNB]) {
#pragma unroll
  for (int c = 0; c < PNB; ++c)
    if (jj + c < nb) psm[(jj + c) * rhp + slot] = xr[c];
}

// MINB = 2 (one row per thread only): capped at 128 registers (~100 bytes of spills) so that two
// CTAs share an SM — large batches run the panels in many waves, and two resident column chains per
// SM hide each other's latency (launch_panel).
template <int RPT, int MINB = 1>
__global__ void __launch_bounds__(PT, MINB) lu_panel_kernel(PanelArgs p) {
  if (p.early) pdl_trigger();
  pdl_wait();   // launched programmatically after the previous chain kernel
  constexpr int SW = 34;
  // one 288-byte message per CTA candidate: shifted live row, value, position
  struct __align__(16) CandMsg {
    double S[SW];
    double val;
    int pos, pad;
  };
  static_assert(sizeof(CandMsg) % 16 == 0, "bulk copies move 16-byte multiples");
  extern __shared__ double psm[];                       // nb columns x rhp slots, then rhp ints
  __shared__ double wval[2][PW];
  __shared__ int wpos[2][PW];
  __shared__ CandMsg cmsg[2][MAXCS];                    // candidates, by source CTA rank
  __shared__ CandMsg cstg[2];                           // local staging of the outgoing message (cs > 1)
  __shared__ __align__(8) uint64_t xbar[2];             // exchange mbarriers (cs > 1)

  const int cs = (int)cluster_nctarank();
  const int rank = (int)cluster_ctarank();
  const int item = blockIdx.x / cs;
  const int n = p.a.n, ld = p.a.ld, nb = p.nb, j0 = p.j0, rhp = p.rhp;
  double* X = p.a.base + (long long)p.slots[item] * p.a.slot_elems;
  int* fpos = reinterpret_cast<int*>(psm + (long long)nb * rhp);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int row_lo = j0 + rank * p.rows_per_cta;
  const int myrows = max(0, min(n, row_lo + p.rows_per_cta) - row_lo);
  const uint32_t xbytes = (uint32_t)cs * (uint32_t)sizeof(CandMsg);
  const double kNaN = __longlong_as_double(0x7ff8000000000000LL);

  for (int e = tid; e < 2 * MAXCS * SW; e += PT) cmsg[e / (MAXCS * SW)][(e / SW) % MAXCS].S[e % SW] = 0.0;
  for (int e = tid; e < 2 * SW; e += PT) cstg[e / SW].S[e % SW] = 0.0;
  if (tid == 0) {
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    fence_barrier_init();
  }

  double x[RPT][PNB];
  int pos[RPT];
  bool valid[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int li = q * PT + tid;
    pos[q] = row_lo + li;
    valid[q] = li < myrows;
#pragma unroll
    for (int c = 0; c < PNB; ++c)
      x[q][c] = (valid[q] && c < nb) ? X[pos[q] + (long long)(j0 + c) * ld] : 0.0;
  }
  // candidate for column 0 (every slot is active)
  double bv = -1.0;
  int bp = INT_MAX;
#pragma unroll
  for (int q = 0; q < RPT; ++q)
    if (valid[q]) {
      const double v = fabs(x[q][0]);
      if (v > bv || (v == bv && pos[q] < bp)) { bv = v; bp = pos[q]; }
    }
  {
    double wv = bv;
    int wi = bp;
    warp_argmax_fast(wv, wi);
    if (lane == 0) { wval[0][warp] = wv; wpos[0][warp] = wi; }
  }
  if (cs > 1) cluster_sync_all(); else __syncthreads();
#ifdef BRI_PANEL_PROFILE
  unsigned long long ph_acc[10] = {0};
  unsigned long long t_last = clock64();
#endif

  for (int jj = 0; jj < nb; ++jj) {
    const int j = j0 + jj;
    const int par = jj & 1;
    if (cs > 1 && tid == 0) mbar_arrive_expect_tx(&xbar[par], xbytes);
    // ---- (1) CTA winner from the warp slots
    double cv = wval[par][lane % PW];
    int cp = wpos[par][lane % PW];
    warp_argmax_fast(cv, cp);
    PPROF(0);
    // ---- (2) stage the CTA candidate; cs > 1: push it to every CTA
    CandMsg* out = cs > 1 ? &cstg[par] : &cmsg[par][0];
    bool mine = false;
    int mq = 0;
#pragma unroll
    for (int q = 0; q < RPT; ++q)
      if (valid[q] && pos[q] == cp) { mine = true; mq = q; }
    if (mine) {
      store_live_row<RPT>(out->S, x, mq);
      out->val = cv;
      out->pos = cp;
    } else if (cp == INT_MAX && tid == 0) {
      out->val = -1.0;
      out->pos = INT_MAX;
    }
    int gp;
    const CandMsg* win;
    if (cs > 1) {
      const bool pub = __any_sync(0xffffffffu, mine) || (cp == INT_MAX && warp == 0);
      if (pub) {
        fence_proxy_async_smem();   // generic smem writes -> visible to the bulk-copy engine
        __syncwarp();
        if (lane < cs)
          bulk_s2cluster(dsmem_addr(&cmsg[par][rank], lane), out, sizeof(CandMsg), dsmem_addr(&xbar[par], lane));
      }
      PPROF(1);
      // CTA-scope acquire: the messages land in this CTA's shared memory
      // through the bulk copies' complete_tx, which orders them; an
      // acquire.cluster here costs a CCTL.IVALL (L1 flush) per column
      mbar_wait(&xbar[par], (jj >> 1) & 1);
      PPROF(2);
      // ---- (3) global winner
      double gv = lane < cs ? cmsg[par][lane].val : -1.0;
      gp = lane < cs ? cmsg[par][lane].pos : INT_MAX;
      const int mypos = gp;
      warp_argmax_fast(gv, gp);
      const int gr = __ffs(__ballot_sync(0xffffffffu, lane < cs && gp != INT_MAX && mypos == gp)) - 1;
      win = &cmsg[par][gr < 0 ? 0 : gr];
    } else {
      PPROF(1);
      __syncthreads();
      PPROF(2);
      gp = cp;
      win = &cmsg[par][0];
    }
    PPROF(3);
    // ---- (4) interchange, scale, rank-1 update
    const bool none = gp == INT_MAX;      // no comparable value in the column: pivot in place
    const int pr = none ? j : gp;
    // plain shared loads through the message pointer: immediate offsets, no
    // per-load address math (the waits above are compiler memory barriers)
    const double* wS = win->S;
    const double piv = none ? kNaN : wS[1];
    if (tid == 0 && rank == 0) p.ipiv[(long long)item * p.n_stride + j] = pr;
    const bool swap = (pr != j && piv != 0.0);  // dgetf2 interchanges only for a nonzero pivot
    const bool recip = fabs(piv) >= kSfmin;
    const double rinv = 1.0 / piv;
    // the finished pivot row: when it is the winning candidate its live values
    // are in the message, and its warp stores the U row with one lane per
    // column; otherwise (zero column pivoted in place) its owner stores it
    int fast_slot = -1;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      if (!valid[q]) continue;
      if (pos[q] == j) {
        if (swap) {
          pos[q] = pr;
        } else if (pr == j && !none) {
          fast_slot = q * PT + tid;
        } else {
          store_u_row(psm, rhp, jj, nb, q * PT + tid, x[q]);
        }
      } else if (swap && pos[q] == pr) {
        pos[q] = j;
        fast_slot = q * PT + tid;
      }
    }
    {
      const unsigned fm = __ballot_sync(0xffffffffu, fast_slot >= 0);
      if (fm) {
        const int slot = __shfl_sync(0xffffffffu, fast_slot, __ffs(fm) - 1);
        if (lane < nb - jj) psm[(jj + lane) * rhp + slot] = wS[lane + 1];
      }
    }
    PPROF(4);
    double u[PNB];
    if (none) {
#pragma unroll
      for (int c = 0; c < PNB; ++c) u[c] = kNaN;
    } else {
#pragma unroll
      for (int c = 0; c < PNB; c += 2) {
        const double2 v = *reinterpret_cast<const double2*>(&wS[c + 2]);
        u[c] = v.x;
        u[c + 1] = v.y;
      }
    }
    double nl[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      nl[q] = 0.0;
      if (!valid[q] || pos[q] <= j) continue;
      double l = x[q][0];
      if (piv != 0.0) l = recip ? l * rinv : l / piv;
      nl[q] = l;
      psm[jj * rhp + q * PT + tid] = l;
      x[q][0] = fma(-l, u[0], x[q][1]);  // next column first
    }
    // next column's candidate + warp reduction (overlaps the remaining updates)
    bv = -1.0;
    bp = INT_MAX;
#pragma unroll
    for (int q = 0; q < RPT; ++q)
      if (valid[q] && pos[q] > j) {
        const double v = fabs(x[q][0]);
        if (v > bv || (v == bv && pos[q] < bp)) { bv = v; bp = pos[q]; }
      }
    {
      double wv = bv;
      int wi = bp;
      warp_argmax_fast(wv, wi);
      if (lane == 0) { wval[par ^ 1][warp] = wv; wpos[par ^ 1][warp] = wi; }
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      if (!valid[q] || pos[q] <= j) continue;
#pragma unroll
      for (int c = 1; c < PNB - 1; ++c) x[q][c] = fma(-nl[q], u[c], x[q][c + 1]);
      x[q][PNB - 1] = 0.0;
    }
    PPROF(5);
    __syncthreads();   // warp slots of the next column complete
  }
#ifdef BRI_PANEL_PROFILE
  if (threadIdx.x == 0 && blockIdx.x == 0)
    for (int k = 0; k < 10; ++k) atomicAdd(&g_panel_phase[k], ph_acc[k]);
#endif

  // write every slot to its final position; publish the interchange map for
  // the rowpanel kernel (position P now holds original row g)
#pragma unroll
  for (int q = 0; q < RPT; ++q)
    if (valid[q]) fpos[q * PT + tid] = pos[q];
  __syncthreads();
  for (int e = tid; e < nb * myrows; e += PT) {
    const int c = e / myrows, i = e % myrows;
    X[fpos[i] + (long long)(j0 + c) * ld] = psm[c * rhp + i];
  }
  int* sig = p.sigma + (long long)item * p.n_stride;
  int* pairs = p.pairs + (long long)item * p.pair_stride + (long long)p.pidx * (1 + 2 * NBMAX);
  for (int i = tid; i < myrows; i += PT) {
    const int P = fpos[i], g = row_lo + i;
    if (P < j0 + nb) {
      sig[P] = g;
    } else if (P != g) {
      const int k = atomicAdd(pairs, 1);
      pairs[1 + 2 * k] = P;
      pairs[2 + 2 * k] = g;
    }
  }
  // no CTA may exit while a peer could still address its shared memory
  if (cs > 1) cluster_sync_all();
}



// ------------------------------------------------------------- tall panel
// Panels taller than the register-resident kernel holds (n - j0 > 8192, e.g.
// b = 20480 of BASELINE config 5): the same dgetf2 decisions with the panel
// kept in global memory (L2-resident: 32 columns x n rows), one 16-CTA cluster
// per factor.  Per column: strided argmax -> warp/CTA/cluster reduction
// (DSMEM stores + cluster barrier) -> physical swap of rows j and p (one
// thread per panel column) -> scale + rank-1 update of the remaining panel
// columns, every thread on its rows.  Three cluster barriers per column;
// slower than the register kernel but unbounded in height.
constexpr int TALL_CS = 16;

struct TallArgs {
  ArenaView a;
  const int* slots;
  int j0, nb, pidx;
  int* ipiv;
  int* sigma;
  int* pairs;
  int* orig;
  int n_stride, pair_stride;
};

__global__ void __launch_bounds__(PT, 1) lu_panel_tall_kernel(TallArgs p) {
  __shared__ double wv[PW];
  __shared__ int wi[PW];
  __shared__ double ws[PW];
  __shared__ double cv[TALL_CS];
  __shared__ double csg[TALL_CS];
  __shared__ int ci[TALL_CS];
  __shared__ int prow;
  __shared__ double psig;
  const int cs = (int)cluster_nctarank();
  const int rank = (int)cluster_ctarank();
  const int item = blockIdx.x / cs;
  const int n = p.a.n, ld = p.a.ld, nb = p.nb, j0 = p.j0;
  double* X = p.a.base + (long long)p.slots[item] * p.a.slot_elems;
  int* orig = p.orig + (long long)item * p.n_stride;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gtid = rank * PT + tid, gthreads = cs * PT;
  for (int i = j0 + gtid; i < n; i += gthreads) orig[i] = i;
  cluster_sync_all();
  for (int jj = 0; jj < nb; ++jj) {
    const int j = j0 + jj;
    double* colj = X + (long long)j * ld;        // X-column j = one memory row
    // ---- argmax |X(i, j)| over i >= j (NaN never wins, smallest index on ties).
    // The SIGNED pivot value travels with its candidate through every level of
    // the reduction: no thread reads X(pr, j) from memory after the winner is
    // known, because rank 0 overwrites that element in the interchange below
    // while lagging CTAs (or warps) could still be reading it.
    double bv = -1.0, bs = 0.0;
    int bi = INT_MAX;
    for (int i = j + gtid; i < n; i += gthreads) {
      const double x = colj[i];
      const double v = fabs(x);
      if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; bs = x; }
    }
    {
      const int mine = bi;
      warp_argmax_fast(bv, bi);
      bs = warp_pick(bs, mine == bi && bi != INT_MAX);
    }
    if (lane == 0) { wv[warp] = bv; wi[warp] = bi; ws[warp] = bs; }
    __syncthreads();
    if (warp == 0) {
      double v = wv[lane % PW], sg = ws[lane % PW];
      int i = wi[lane % PW];
      const int mine = i;
      warp_argmax_fast(v, i);
      sg = warp_pick(sg, mine == i && i != INT_MAX);
      if (lane < cs) {   // our CTA's candidate into slot `rank` of every CTA
        const uint32_t a = dsmem_addr(&cv[rank], lane), b = dsmem_addr(&ci[rank], lane);
        const uint32_t c = dsmem_addr(&csg[rank], lane);
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
        asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(b), "r"(i) : "memory");
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(c), "d"(sg) : "memory");
      }
    }
    cluster_sync_all();
    if (warp == 0) {
      double v = lane < cs ? cv[lane] : -1.0, sg = lane < cs ? csg[lane] : 0.0;
      int i = lane < cs ? ci[lane] : INT_MAX;
      const int mine = i;
      warp_argmax_fast(v, i);
      sg = warp_pick(sg, mine == i && i != INT_MAX);
      if (lane == 0) {
        prow = (i == INT_MAX) ? j : i;   // all NaN: pivot in place (no interchange)
        psig = sg;
      }
    }
    __syncthreads();
    const int pr = prow;
    // all-NaN column: pr == j, nothing is swapped, so X(j, j) is stable to read
    const double piv = (pr == j) ? colj[j] : psig;
    if (tid == 0 && rank == 0) p.ipiv[(long long)item * p.n_stride + j] = pr;
    const bool swap = (pr != j && piv != 0.0);
    if (swap && rank == 0) {
      if (tid < nb) {
        double* col = X + (long long)(j0 + tid) * ld;
        const double t = col[j];
        col[j] = col[pr];
        col[pr] = t;
      } else if (tid == nb) {
        const int t = orig[j];
        orig[j] = orig[pr];
        orig[pr] = t;
      }
    }
    cluster_sync_all();   // the interchange is visible cluster-wide (release / acquire)
    // ---- scale and rank-1 update of columns jj+1.. on rows i > j
    const bool recip = fabs(piv) >= kSfmin;
    const double rinv = 1.0 / piv;
    double u[NBMAX];   // the pivot row's remaining panel entries (same for every row)
#pragma unroll
    for (int c = 0; c < NBMAX; ++c) u[c] = (c > jj && c < nb) ? X[(long long)(j0 + c) * ld + j] : 0.0;
    for (int i = j + 1 + gtid; i < n; i += gthreads) {
      double l = colj[i];
      if (piv != 0.0) {
        l = recip ? l * rinv : l / piv;
        colj[i] = l;
      }
      double v[NBMAX];   // all loads of the row first: one L2 round trip, not one per column
#pragma unroll
      for (int c = 0; c < NBMAX; ++c)
        if (c > jj && c < nb) v[c] = X[(long long)(j0 + c) * ld + i];
#pragma unroll
      for (int c = 0; c < NBMAX; ++c)
        if (c > jj && c < nb) X[(long long)(j0 + c) * ld + i] = fma(-l, u[c], v[c]);
    }
    cluster_sync_all();   // column jj+1 is final before its argmax
  }
  // position P in [j0, n) now holds original row orig[P]
  int* sig = p.sigma + (long long)item * p.n_stride;
  int* pairs = p.pairs + (long long)item * p.pair_stride + (long long)p.pidx * (1 + 2 * NBMAX);
  for (int P = j0 + gtid; P < n; P += gthreads) {
    const int g = orig[P];
    if (P < j0 + nb) {
      sig[P] = g;
    } else if (g != P) {
      const int k = atomicAdd(pairs, 1);
      pairs[1 + 2 * k] = P;
      pairs[2 + 2 * k] = g;
    }
  }
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
  int early;          // pdl_trigger before the wait (bri_internal.h)
  int compose_pi;     // this launch folds the panel's interchanges into pi (exactly one launch per panel does)
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
  if (p.early) pdl_trigger();
  pdl_wait();
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
    if (!p.compose_pi) return;
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

// ------------------------------------------------------------- deferred interchanges
// snap[item][J][pi[x]] = x: where each original row sat after outer block J
__global__ void pi_snapshot_kernel(const int* pi, int* snap, int n, int nob, int J) {
  const int item = blockIdx.x;
  const int* p = pi + (long long)item * n;
  int* q = snap + ((long long)item * nob + J) * n;
  for (int x = threadIdx.x; x < n; x += blockDim.x) q[p[x]] = x;
}

constexpr int LD_WARPS = 8;
constexpr int LD_MAXN = 2048;   // orders it handles: 8 column segments (< n doubles) + the composed map fit in smem

// All L columns of outer block J (rows >= (J+1)*outer) of one factor, one CTA: the composed map
// src(x) = inv_J[pi[x]] (where the row now at final position x sat after block J) is built once
// in smem, then each warp reorders its columns through a staged copy — the interchanges of every
// later block at once, two coalesced passes per column.
__global__ void __launch_bounds__(LD_WARPS * 32) laswp_deferred_kernel(ArenaView a, const int* slots,
                                                                       const int* pi, const int* snap,
                                                                       int nob, int outer, int ncols) {
  extern __shared__ double seg_s[];
  const int n = a.n;
  int* comp = reinterpret_cast<int*>(seg_s + (long long)LD_WARPS * n);   // smem sized by n at launch
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int J = blockIdx.x, item = blockIdx.y;
  const int r0 = (J + 1) * outer;
  const int* p = pi + (long long)item * n;
  const int* inv = snap + ((long long)item * nob + J) * n;
  for (int x = r0 + threadIdx.x; x < n; x += blockDim.x) comp[x - r0] = inv[p[x]] - r0;
  __syncthreads();
  double* seg = seg_s + (long long)warp * n;
  const int c_end = min((J + 1) * outer, ncols);
  for (int c = J * outer + warp; c < c_end; c += LD_WARPS) {
    double* col = a.base + (long long)slots[item] * a.slot_elems + (long long)c * a.ld;
    for (int x = r0 + lane; x < n; x += 32) seg[x - r0] = col[x];
    __syncwarp();
    for (int x = r0 + lane; x < n; x += 32) col[x] = seg[comp[x - r0]];
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
  unsigned long long z[10] = {0};
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
                            int pi_stride, bool identity_src, cudaStream_t s, const int* pidx) {
  const int gx = a.n < 512 ? a.n : 512;
  count_launch();
  permcopy_kernel<<<dim3(gx, count), 256, 0, s>>>(a, pairs, pi, pi_stride, identity_src ? 1 : 0, pidx);
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

cudaError_t launch_pi_init(int* pi, int n, int count, unsigned long long* scale_bits, int* pairs, int pair_stride,
                           cudaStream_t s) {
  count_launch();
  const int work = n > pair_stride ? n : pair_stride;
  pi_init_kernel<<<dim3((work + 255) / 256, count), 256, 0, s>>>(pi, n, scale_bits, pairs, pair_stride);
  return cudaGetLastError();
}

// Panel width: 32 columns, held in registers (up to 2 rows x 32 per thread).
int panel_width(int n) { return n > 0 ? NBMAX : NBMAX; }

template <int RPT, int MINB = 1>
static cudaError_t launch_panel_t(PanelArgs p, int cs, int count, cudaStream_t s) {
  const size_t smem = (size_t)p.nb * p.rhp * 8 + (size_t)p.rhp * 4 + 16;
  if (smem > 160 * 1024) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(count * cs);
  cfg.blockDim = dim3(PT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  pdl_attr(attr[1]);
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  count_launch();
  return cudaLaunchKernelEx(&cfg, lu_panel_kernel<RPT, MINB>, p);
}

cudaError_t configure_lu() {
  cudaError_t e = cudaFuncSetAttribute(lu_panel_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(lu_panel_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(lu_panel_kernel<1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(lu_panel_kernel<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(lu_panel_kernel<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(lu_panel_tall_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(laswp_deferred_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             LD_WARPS * LD_MAXN * 8 + LD_MAXN * 4);
  return e;
}

int max_panel_rows() { return MAXCS * 2 * PT; }

cudaError_t launch_panel(const ArenaView& a, const int* slots, int count, int j0, int nb, int pidx,
                         const LuScratch& sc, int n_stride, int pair_stride, cudaStream_t s, bool early) {
  const int h = a.n - j0;
  // 1 row per thread while it fits a cluster of 8, else 2 (registers: 2 x 32 doubles)
  // Up to 8 x PT rows: 1 row per thread, portable clusters (measured: beats a
  // halved cluster at 2 rows); up to 8 x 2 x PT: 2 rows; beyond, 16-CTA clusters.
  // (one row per thread on a 16-CTA cluster is faster alone at 4096 rows — 1.70
  // vs 1.87 us/column — but a 16-SM cluster waits for SMs next to the
  // concurrent trailing update: config 2 went from 35.0 to 39.4 ms)
  // BRI_TALL_ROWS lowers the tall-panel threshold (tests and compute-sanitizer runs
  // exercise the tall kernel on small matrices); default: what registers cannot hold
  static const int tall_rows = [] {
    const char* e = getenv("BRI_TALL_ROWS");
    return e ? atoi(e) : max_panel_rows();
  }();
  if (h > tall_rows) {
    TallArgs t{a, slots, j0, nb, pidx, sc.ipiv, sc.sigma, sc.pairs, sc.orig, n_stride, pair_stride};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(count * TALL_CS);
    cfg.blockDim = dim3(PT);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = TALL_CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    count_launch();
    return cudaLaunchKernelEx(&cfg, lu_panel_tall_kernel, t);
  }
  // Large batches run in many waves of one CTA per SM (registers bound the rows
  // resident per SM), so beyond two waves two rows per thread halves the waves
  // (config 3: 1.60 -> 1.52 s).
  static const int wide_waves = [] {
    const char* e = getenv("BRI_PANEL_RPT2_WAVES");
    return e ? atoi(e) : 2;
  }();
  // BRI_PANEL_2CTA=1: instead, keep one row per thread and run two CTAs per SM (128 registers)
  static const int two_cta = [] {
    const char* e = getenv("BRI_PANEL_2CTA");
    return e ? atoi(e) : 0;
  }();
  int rpt = h <= PORTABLE_CS * PT ? 1 : 2;
  bool dense = false;
  if (rpt == 1 && h > PT) {
    const long long ctas1 = (long long)count * ((h + PT - 1) / PT);
    if (ctas1 > (long long)wide_waves * 148) {
      if (two_cta) dense = true;
      else rpt = 2;
    }
  }
  int cs = 1;
  while (cs < MAXCS && (h + cs - 1) / cs > rpt * PT) cs <<= 1;
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
  p.early = early ? 1 : 0;
  if (dense && (size_t)p.nb * p.rhp * 8 + (size_t)p.rhp * 4 + 16 <= 100 * 1024) return launch_panel_t<1, 2>(p, cs, count, s);
  if (rpt == 1) return launch_panel_t<1>(p, cs, count, s);
  return launch_panel_t<2>(p, cs, count, s);
}

cudaError_t launch_rowpanel(const ArenaView& a, const int* slots, int count, int j0, int nb, int pidx,
                            int cbeg, int cend, const LuScratch& sc, int n_stride, int pair_stride,
                            cudaStream_t s, bool compose_pi, bool early) {
  RowPanelArgs p;
  p.compose_pi = compose_pi ? 1 : 0;
  p.early = early ? 1 : 0;
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
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(gx, count);
  cfg.blockDim = dim3(RP_THREADS);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  pdl_attr(attr[0]);
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  count_launch();
  return cudaLaunchKernelEx(&cfg, rowpanel_kernel, p);
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

int laswp_deferred_max_n() { return LD_MAXN; }

cudaError_t launch_pi_snapshot(const int* pi, int* snap, int n, int nob, int J, int count, cudaStream_t s) {
  count_launch();
  pi_snapshot_kernel<<<count, 256, 0, s>>>(pi, snap, n, nob, J);
  return cudaGetLastError();
}

cudaError_t launch_laswp_deferred(const ArenaView& a, const int* slots, int count, const int* pi,
                                  const int* snap, int nob, int outer, cudaStream_t s) {
  const int ncols = (nob - 1) * outer;   // the last block has no later interchanges
  if (ncols <= 0) return cudaSuccess;
  count_launch();
  const int smem = LD_WARPS * a.n * 8 + a.n * 4;
  laswp_deferred_kernel<<<dim3(nob - 1, count), LD_WARPS * 32, smem, s>>>(
      a, slots, pi, snap, nob, outer, ncols);
  return cudaGetLastError();
}

cudaError_t launch_diag_check(const ArenaView& a, const int* slots, int count,
                              const unsigned long long* scale_bits, int* status, cudaStream_t s) {
  count_launch();
  diag_check_kernel<<<count, 256, 0, s>>>(a, slots, scale_bits, status);
  return cudaGetLastError();
}

}  // namespace bri
