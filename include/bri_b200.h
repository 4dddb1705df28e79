/*
 * bri_b200.h — C ABI of the B200 BRI hot path (libbri_b200.so).
 *
 * The reference (`bri`, pure Python) has no FFI of its own: its hot path calls
 * numpy/scipy, i.e. OpenBLAS dgemm and LAPACK dgetrf/dgetrs, from
 *   pkg/src/bri/core.py:173-181   multiply      (x @ y)
 *   pkg/src/bri/core.py:184-197   subtract      (x -= y)
 *   pkg/src/bri/core.py:238-263   invert_dense  (dgetrf on x.T, pivot test, dgetrs vs I)
 *   pkg/src/bri/core.py:212-235   lu_factor     (dgetrf on x)
 *   pkg/src/bri/engine.py:157-180 _fold         (r - l @ (inv(p) @ rt) per Schur node)
 * The entry points below are what a maintainer binds in place of those calls
 * (ctypes stub in INTEGRATION.md).  Plain pointers and sizes only; all buffers
 * are caller-owned device memory; nothing throws across the ABI.
 *
 * Memory model: an *arena* is caller-owned device memory holding `nslots`
 * blocks of order n, slot s at base + s * n * ld doubles, each block stored
 * row-major with row stride ld (ld % 8 == 0, ld >= n) — i.e. exactly the bytes
 * of the reference's C-ordered (b, b) float64 ndarray.  Kernels read a slot as
 * the column-major transpose (the LAPACK view the reference factors,
 * core.py:249).  Items name slots by index.
 *
 * Return value: 0 on success, < 0 on a CUDA / argument error
 * (bri_last_error() has the message).  Singular pivots are NOT errors at this
 * level: they are reported per item in `status` (0 = ok, otherwise the 1-based
 * index of the first pivot with |u_ii| <= n * eps * max|A|, NaN flagged), the
 * caller maps them to SingularBlockError / SingularPivotError
 * (errors.py:26-69) as the reference does.
 */
#ifndef BRI_B200_H
#define BRI_B200_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bri_ctx bri_ctx;
typedef struct bri_arena bri_arena;

/* ABI version (major * 100 + minor). */
int bri_version(void);

/* Number of kernels this library has launched in the process so far. */
long long bri_launch_count(void);

/* Executed FLOPs this library has issued so far, per kernel family
 * (0: GEMM kernels, 2*M*N*K per item; 1: triangular-solve leaves); -1 for a bad kind.
 * Graph replays count what their kernels execute. */
long long bri_flop_count(int kind);

/* Message of the last failed call on this thread ("" if none). */
const char* bri_last_error(void);

/* Per-device context: kernel attributes, staging buffers, TMA encoder. */
int bri_ctx_create(int device, bri_ctx** out);
void bri_ctx_destroy(bri_ctx* ctx);

/* Wrap caller-owned device memory as an arena (builds the TMA descriptors). */
int bri_arena_create(bri_ctx* ctx, double* base, int n, int ld, int nslots, bri_arena** out);
void bri_arena_destroy(bri_arena* arena);

/*
 * Schur nodes, batched — replaces engine.py:157-180 (_fold) for `count` nodes.
 * items: 7 ints per node: slots (p, rt, l, r, out, f, w); f and w are scratch
 * slots (f receives the LU factors of p, w the solve).  Computes, per node,
 *     out = r - l @ inv(p) @ rt          (row-major block semantics)
 * with 1 factorization + 1 solve + 1 fused GEMM-subtract.  p/rt/l/r are not
 * modified (out may alias r).  status (device, count ints): pivot test of p.
 */
int bri_schur_batch(bri_arena* arena, void* stream, int count, const int* items, int* status);

/*
 * One level of the deduplicated DAG with its shared work factored out —
 * replaces engine.py:157-180 (_fold) for every node of the level.
 *   fitems: nf pairs (p, F): F <- LU factors of p (dgetrf on the column-major view,
 *           core.py:249); fstatus (device, nf ints): pivot test of p (core.py:200-209).
 *   sitems: ns triples (f, l, W): W <- solve with factor f (0-based index into fitems)
 *           of the right-hand side l (dgetrs, core.py:259), i.e. inv(p) applied to l.
 *   gitems: ng quads (rt, W, r, out): out = r - rt (X) W (multiply + subtract,
 *           core.py:173-197; out may alias r).
 * In row-major block semantics each node's result is r - l @ inv(p) @ rt.
 * Orders <= 96 are rejected (bri_schur_batch handles them in one kernel).
 */
int bri_level_batch(bri_arena* arena, void* stream, int nf, const int* fitems, int ns, const int* sitems, int ng,
                    const int* gitems, int* fstatus);

/*
 * bri_level_batch whose operands may still be in flight (the first DAG level of
 * a run fed from pinned host memory): the caller's stream must already wait for
 * the pivots; the solves wait on ev_l (cudaEvent_t, l operands landed) and the
 * GEMM-subtracts on ev_rtr (rt and r landed).  Either event may be NULL.
 */
int bri_level_batch_gated(bri_arena* arena, void* stream, int nf, const int* fitems, int ns, const int* sitems,
                          int ng, const int* gitems, int* fstatus, void* ev_l, void* ev_rtr);

/*
 * The general level batch: as bri_level_batch_gated, plus right-side solves for
 * pivots whose nodes share fewer distinct rt than l operands (the reference's own
 * association (rt · inv(p)) · l, engine.py:167-174, in X-world): C = rt^ p^-1 solved once
 * per distinct (pivot, rt), then out = r - C * l.  titems: 2 ints (factor index into
 * fitems, Ft scratch slot) per factor used on that side; ritems: 4 ints (index into
 * titems, rt slot, S scratch slot, C output slot); GEMM items of those nodes are
 * (C, l, r, out).  nt = nr = 0 is bri_level_batch_gated.
 */
int bri_level_batch_ex(bri_arena* arena, void* stream, int nf, const int* fitems, int ns, const int* sitems,
                       int nt, const int* titems, int nr, const int* ritems, int ng, const int* gitems, int* fstatus,
                       void* ev_l, void* ev_rtr);

/*
 * A whole small-order DAG run (order <= 96, e.g. BASELINE config 1) in one call and one
 * CUDA graph — replaces the per-level bri_schur_batch + bri_invert_batch sequence for the
 * reference's reduce_frame / invert_block recursion (engine.py:196-273) on an HBM-resident M:
 * gitems (block row, block col, slot) gathered from the row-major device matrix M (leading
 * dim ldm); nlev levels of lev_counts[l] nodes, nitems 5 ints each (p, rt, l, r, out) in
 * level order, node_status one int per node; ninv final inversions, iitems (in, out),
 * inv_status one int each.  Statuses as bri_schur_batch / bri_invert_batch.
 */
int bri_dag_small(bri_arena* arena, void* stream, const double* M, long long ldm, int ng, const int* gitems,
                  int nlev, const int* lev_counts, const int* nitems, int* node_status, int ninv,
                  const int* iitems, int* inv_status);

/*
 * Block inverses, batched — replaces core.py:238-263 (invert_dense).
 * items: 3 ints per block: slots (in, f, out); f is scratch; in is not modified.
 * status (device, count ints): pivot test of in.
 */
int bri_invert_batch(bri_arena* arena, void* stream, int count, const int* items, int* status);

/*
 * LU with partial pivoting in place, batched — dgetrf semantics on the
 * column-major view of each slot (i.e. on the transpose of the row-major
 * block, as core.py:249).  perm (device, count * n ints, may be NULL):
 * 0-based row permutation, (P X)[x] = X[perm[x]].  ipiv (device, count * n,
 * may be NULL): LAPACK-style 0-based interchanges.  status as above.
 */
int bri_getrf_batch(bri_arena* arena, void* stream, int count, const int* slots, int* ipiv,
                    int* perm, int* status);

/*
 * Solve with LU factors, batched — dgetrs(trans = 'N') semantics on the
 * column-major views (core.py:259): dst = X^-1 * src where X's factors are in
 * slot f (from bri_getrf_batch) and perm its row permutation (device, count * n).
 * items: 3 ints (f, src, dst), dst != src.
 */
int bri_getrs_batch(bri_arena* arena, void* stream, int count, const int* items, const int* perm);

/*
 * GEMM, batched — replaces core.py:173-181 (multiply) fused with
 * core.py:184-197 (subtract).  Column-major window semantics on each slot:
 *   C_out[c_r0:+M, c_c0:+N] = beta * C_in[...] + alpha * A[a_r0:+M, a_c0:+K] * B[b_r0:+K, b_c0:+N]
 * items: 4 ints per product: slots (A, B, C_in, C_out).  For row-major blocks
 * x @ y pass A = y, B = x.  beta == 0 never reads C_in.  a_r0 and b_r0 (the
 * contiguous-dimension offsets) must be even: TMA boxes start 16-byte aligned.
 */
int bri_gemm(bri_arena* arena, void* stream, int count, const int* items, int M, int N, int K,
             int a_r0, int a_c0, int b_r0, int b_c0, int c_r0, int c_c0, double alpha,
             double beta);

/* out = alpha * x + beta * y elementwise over whole slots; items: (x, y, out). */
int bri_axpby(bri_arena* arena, void* stream, int count, const int* items, double alpha,
              double beta);

/* out = transpose(src) over whole slots; items: (src, out), out != src. */
int bri_transpose(bri_arena* arena, void* stream, int count, const int* items);

/*
 * Block gather — replaces the per-fetch copy of providers.py:318-336 +
 * core.py:92-98 for a matrix resident in device memory.  M: dense row-major
 * device matrix with leading dim ldm (elements); items: 3 ints per block
 * (block row i, block col j, destination slot), 0-based, block order = arena n.
 */
int bri_gather_blocks(bri_arena* arena, void* stream, const double* M, long long ldm, int count,
                      const int* items);

/*
 * Element gather for padded layouts — replaces the shifted-window fetch of
 * providers.py:203-271,380-402.  Block (i, j) of the view (0-based, order n =
 * arena order) is [[M, 0], [0, I]] (M: m x m row-major device matrix, leading
 * dim ldm) at element rows rmap[i*n .. i*n+n) and columns cmap[j*n .. j*n+n)
 * (device int arrays of length k*n).  items: 3 ints (i, j, destination slot).
 */
int bri_gather_elements(bri_arena* arena, void* stream, const double* M, long long ldm, int m,
                        const int* rmap, const int* cmap, int count, const int* items);

/*
 * LS-SVM kernel system matrix generated on the device — replaces the
 * per-fetch element evaluation of providers.py:175-200 (_KernelSource.rect,
 * KernelSpec providers.py:93-120).  x: n x d row-major device inputs; the
 * matrix has order m = n + 1: (0,0) = 0, the rest of row/column 0 = 1,
 * interior (i, j) = exp(sq_ij / denom) + (i == j ? ridge : 0) with sq_ij the
 * squared distance of inputs i-1 and j-1 summed in numpy's pairwise order,
 * denom = -2 sigma^2 and ridge = 1 / gamma as the caller computes them.
 * Indices >= m are the identity padding of [[M, 0], [0, I]].
 *
 * bri_rbf_blocks writes view blocks (i, j) of order n_arena into slots —
 * items: 3 ints (block row, block col, slot), 0-based — with element rows
 * rmap[i*n_arena + r] and columns cmap[j*n_arena + c] (device int arrays, or
 * both NULL for the identity view).  bri_rbf_dense writes the whole m x m
 * matrix row-major into out (leading dim ldo >= m).
 */
int bri_rbf_blocks(bri_arena* arena, void* stream, const double* x, int n, int d, double denom, double ridge,
                   const int* rmap, const int* cmap, int count, const int* items);
int bri_rbf_dense(void* stream, const double* x, int n, int d, double denom, double ridge, double* out,
                  long long ldo);

/*
 * Seeded Gaussian test matrix M = G + shift * I of order m, generated blockwise
 * on the device (BASELINE config 5: "M = G + m I, G i.i.d. N(0,1) generated
 * blockwise from seed 4"; the reference has no blockwise scheme, it draws the
 * whole matrix from one PCG64 stream, cli.py:122-130).  Element (r, c) takes
 * Philox4x64-10 (numpy's np.random.Philox) at counter ((r*m + c) / 4, 0, 0, 0)
 * with key (seed, 0), then Box-Muller on the output pair (r*m + c) % 4 / 2
 * (cos for even, sin for odd r*m + c).  Indices >= m are identity padding.
 * bri_randn_blocks writes view blocks (i, j) of order n_arena into slots
 * (items as bri_rbf_blocks, optional rmap/cmap); bri_randn_window writes the
 * rows x cols window at (row0, col0) row-major into out (leading dim ldo).
 */
int bri_randn_blocks(bri_arena* arena, void* stream, long long m, unsigned long long seed, double shift,
                     const int* rmap, const int* cmap, int count, const int* items);
int bri_randn_window(void* stream, long long m, unsigned long long seed, double shift, long long row0,
                     long long col0, int rows, int cols, double* out, long long ldo);

/*
 * Device -> host store of a result block — the output side of sink.put
 * (formats.py:249-282): one 2-D async copy of rows x cols doubles from a
 * row-major device buffer (leading dim ldd) into a row-major host canvas
 * (leading dim ldh).  With a pinned canvas the copy is asynchronous on
 * `stream`; the caller synchronizes before reading the canvas.
 */
int bri_store_host(void* stream, double* host, long long ldh, const double* dev, long long ldd, int rows,
                   int cols);

/*
 * Host -> device block loads — the fetch of providers.py:318-336 for a matrix in
 * (pinned) host memory: one 2-D async copy per item (block row i, block col j,
 * slot), 0-based, from the row-major host matrix with leading dim ldh into the
 * slot's row-major b x b window.  Pinned host memory keeps the copies
 * asynchronous on `stream`.
 */
int bri_load_host_blocks(bri_arena* arena, void* stream, const double* host, long long ldh, int count,
                         const int* items);

/*
 * bri_schur_batch with input gates: the stream waits on ev_l (an event, may be
 * NULL) before reading the l operands and on ev_rtr before reading rt and r,
 * so the pivot factorization overlaps the copies of the other operands.  The
 * p operands must be resident when the call is issued.  Not graph-captured.
 */
int bri_schur_batch_gated(bri_arena* arena, void* stream, int count, const int* items, int* status, void* ev_l,
                          void* ev_rtr);

/* FP64 DMMA throughput probe (register-only mma.sync loop on every SM);
 * writes achieved TFLOP/s.  Used by bench.py as the roofline denominator. */
int bri_fp64_peak(void* stream, int iters, double* tflops);

#ifdef __cplusplus
}
#endif

#endif /* BRI_B200_H */
