// C ABI of libbri_b200.so (include/bri_b200.h): contexts, arenas (TMA
// descriptors over caller-owned device memory) and the batched hot-path
// operations that stand in for the reference's BLAS/LAPACK calls.
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX: free unless a profiler is attached

#include "../../include/bri_b200.h"
#include "bri_common.cuh"
#include "bri_internal.h"

using namespace bri;

namespace bri {
static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
// Executed-FLOP ledger per kernel family (FLOP_GEMM: gemm/skinny/persistent
// GEMM kernels, FLOP_TRSM: triangular-solve leaves): the numerator bench.py
// divides by the family's in-step kernel time for the roofline.  Graph
// replays add what their capture recorded (thread-local capture delta).
static std::atomic<long long> g_flops[FLOP_KINDS];
static thread_local long long tl_flops[FLOP_KINDS];
void count_flops(int kind, double f) {
  const long long v = (long long)f;
  g_flops[kind].fetch_add(v, std::memory_order_relaxed);
  tl_flops[kind] += v;
}
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("BRI_PDL");
    return e == nullptr || e[0] != '0';
  }();
  return on;
}
}  // namespace bri

namespace {

thread_local std::string g_last_error;

int fail(const char* what, cudaError_t e) {
  g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return -1;
}

int fail_msg(const std::string& msg) {
  g_last_error = msg;
  return -2;
}

#define BRI_CHECK(call)                          \
  do {                                           \
    cudaError_t _e = (call);                     \
    if (_e != cudaSuccess) return fail(#call, _e); \
  } while (0)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encoder() {
  static EncodeTiledFn fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// Grow-only device buffer whose reuse is ordered by the (single) stream a
// context is driven from.
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  int ensure(size_t need, cudaStream_t s) {
    if (need <= bytes) return 0;
    size_t nb = need + need / 2 + 4096;
    if (ptr != nullptr) BRI_CHECK(cudaFreeAsync(ptr, s));
    ptr = nullptr;
    BRI_CHECK(cudaMallocAsync(&ptr, nb, s));
    bytes = nb;
    return 0;
  }
};

}  // namespace

struct GraphEntry {
  std::vector<uintptr_t> key;
  cudaGraphExec_t exec;
  long long kernels;  // kernel nodes: counted as launches on every replay
  long long flops[FLOP_KINDS];   // executed FLOPs per family: counted on every replay
};

struct bri_ctx {
  int device = 0;
  cudaStream_t side = nullptr;    // lookahead: bulk trailing updates of the LU
  cudaStream_t side2 = nullptr;   // folded right-hand side of the Schur LU (LuFold)
  cudaStream_t side3 = nullptr;   // a block's first inner panel carried on to the next block's columns
  cudaStream_t gstream = nullptr; // graphs are captured / launched here
  cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_x = nullptr, ev_d = nullptr, ev_w = nullptr;
  cudaEvent_t ev_p = nullptr, ev_y = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  std::vector<GraphEntry> graphs; // captured hot-path sequences (LRU, <= 16)
  std::vector<std::vector<uintptr_t>> seen;
  DevBuf items;   // uploaded item arrays
  DevBuf lu;      // LU scratch
  DevBuf dinv;    // inverted diagonal blocks of L and U (fused triangular solves)
  std::vector<int> host;  // staging for item arrays
  // pinned staging ring for item uploads: a pageable source would make
  // cudaMemcpyAsync wait for the stream to drain, so the host could not
  // submit the next (large) graph while the GPU still runs the previous work
  static constexpr int NSTAGE = 4;
  void* stage[NSTAGE] = {};
  size_t stage_bytes[NSTAGE] = {};
  cudaEvent_t stage_ev[NSTAGE] = {};
  int stage_next = 0;
};

struct bri_arena {
  bri_ctx* ctx = nullptr;
  ArenaView v{};
  alignas(64) CUtensorMap tmA;
  alignas(64) CUtensorMap tmB;
  alignas(64) CUtensorMap tmB32;
  alignas(64) CUtensorMap tmB16;
};

namespace {

// ---------------------------------------------------------------- helpers
// Upload `words` host ints into the context's device buffer (stream-ordered).
int upload(bri_ctx* ctx, cudaStream_t s, const std::vector<int>& h, int** dev) {
  const size_t bytes = h.size() * sizeof(int);
  if (int rc = ctx->items.ensure(bytes, s)) return rc;
  const int k = ctx->stage_next;
  ctx->stage_next = (k + 1) % bri_ctx::NSTAGE;
  if (ctx->stage_ev[k] == nullptr) {
    BRI_CHECK(cudaEventCreateWithFlags(&ctx->stage_ev[k], cudaEventDisableTiming));
  } else {
    BRI_CHECK(cudaEventSynchronize(ctx->stage_ev[k]));   // its previous copy has been read
  }
  if (ctx->stage_bytes[k] < bytes) {
    if (ctx->stage[k] != nullptr) BRI_CHECK(cudaFreeHost(ctx->stage[k]));
    ctx->stage[k] = nullptr;
    const size_t nb = bytes + bytes / 2 + 4096;
    BRI_CHECK(cudaHostAlloc(&ctx->stage[k], nb, cudaHostAllocDefault));
    ctx->stage_bytes[k] = nb;
  }
  std::memcpy(ctx->stage[k], h.data(), bytes);
  BRI_CHECK(cudaMemcpyAsync(ctx->items.ptr, ctx->stage[k], bytes, cudaMemcpyHostToDevice, s));
  BRI_CHECK(cudaEventRecord(ctx->stage_ev[k], s));
  *dev = static_cast<int*>(ctx->items.ptr);
  return 0;
}

int env_or(const char* name, int dflt) {
  const char* e = getenv(name);
  return (e && *e) ? atoi(e) : dflt;
}

struct LuLayout {
  int n, count, npanels, pair_stride;
  size_t off_ipiv, off_pi, off_sigma, off_pairs, off_scale, off_status, off_orig, off_snap, total;
};

LuLayout lu_layout(int n, int count) {
  LuLayout L;
  L.n = n;
  L.count = count;
  const int nb = panel_width(n);
  L.npanels = (n + nb - 1) / nb;
  L.pair_stride = L.npanels * (1 + 2 * NBMAX);
  size_t off = 0;
  auto take = [&](size_t b) {
    size_t o = off;
    off += (b + 255) & ~size_t(255);
    return o;
  };
  L.off_ipiv = take((size_t)count * n * 4);
  L.off_pi = take((size_t)count * n * 4);
  L.off_sigma = take((size_t)count * n * 4);
  L.off_pairs = take((size_t)count * L.pair_stride * 4);
  L.off_scale = take((size_t)count * 8);
  L.off_status = take((size_t)count * 4);
  L.off_orig = take((size_t)count * n * 4);
  L.off_snap = n <= laswp_deferred_max_n() ? take((size_t)count * ((n + LU_OUTER - 1) / LU_OUTER) * n * 4) : off;
  L.total = off;
  return L;
}

LuScratch lu_scratch(void* base, const LuLayout& L) {
  char* b = static_cast<char*>(base);
  LuScratch s;
  s.ipiv = reinterpret_cast<int*>(b + L.off_ipiv);
  s.pi = reinterpret_cast<int*>(b + L.off_pi);
  s.sigma = reinterpret_cast<int*>(b + L.off_sigma);
  s.pairs = reinterpret_cast<int*>(b + L.off_pairs);
  s.scale_bits = reinterpret_cast<unsigned long long*>(b + L.off_scale);
  s.status = reinterpret_cast<int*>(b + L.off_status);
  s.orig = reinterpret_cast<int*>(b + L.off_orig);
  s.snap = reinterpret_cast<int*>(b + L.off_snap);
  return s;
}

int gemm_call(bri_arena* ar, cudaStream_t s, const int* dev_items, int count, int M, int N, int K,
              int a_r0, int a_c0, int b_r0, int b_c0, int c_r0, int c_c0, double alpha, double beta,
              int max_ctas = 0, int overlap = 0, int early = 0) {
  GemmParams p{};
  p.early = early;
  p.max_ctas = max_ctas;
  p.overlap = overlap;
  p.base = ar->v.base;
  p.ld = ar->v.ld;
  p.slot_elems = ar->v.slot_elems;
  p.items = dev_items;
  p.M = M;
  p.N = N;
  p.K = K;
  p.a_r0 = a_r0;
  p.a_c0 = a_c0;
  p.b_r0 = b_r0;
  p.b_c0 = b_c0;
  p.c_r0 = c_r0;
  p.c_c0 = c_c0;
  p.alpha = alpha;
  p.beta = beta;
  count_flops(FLOP_GEMM, 2.0 * M * N * (double)K * count);
  // tuning aid (BRI_GEMM_LOG=1): the shapes the solver issues, in capture order
  static const bool log_shapes = [] { const char* e = getenv("BRI_GEMM_LOG"); return e && *e == '1'; }();
  if (log_shapes) fprintf(stderr, "GEMMLOG %d %d %d %d %d\n", M, N, K, count, max_ctas);
  BRI_CHECK(launch_gemm(ar->tmA, ar->tmB, ar->tmB32, p, count, s));
  return 0;
}

// Blocked right-looking LU (dgetrf) of `count` slots in place, two levels
// with lookahead:
//   * outer blocks of 128 columns, each factored by 32-wide inner panels
//     (cluster panel kernel + rowpanel + rank-32 GEMM);
//   * batches of <= 2 (panel chain = critical path): the inner panels of
//     block J also carry the NEXT block's 128 columns (interchanges, 32-row
//     solve and rank-32 update per inner panel), so block J+1 is ready the
//     moment block J's last panel finishes; meanwhile the side stream applies
//     block J's interchanges / U12 solve / rank-128 update to block J+2's
//     columns first (an event the main stream waits on before its own inner
//     panels reach them), then to everything else;
//   * larger batches: block J's update is applied first to block J+1's
//     columns on the caller's stream, which then factors block J+1 while the
//     side stream updates everything else.
//   Either way the pivot chain (panels) overlaps the bulk trailing GEMMs.
// dev_slots: F slots; dev_ffff: (F, F, F, F) quads; dev_ff: (F, F) pairs.
//
// fold: a forward sweep rides along as extra columns of the factorization,
// on a second side stream that trails the panels, so only the U sweep is
// left after the factorization.  The left-of-block interchanges of L are
// skipped then (nothing reads the final L).
//   * Schur nodes: W = L^-1 P l — W <- l, then per outer block J its
//     interchanges, the L11 solve of J's rows and the rank-128 update of the
//     rows below;
//   * explicit inverses (tri): W = L^-1 itself — W <- I; per block J the
//     interchanges of W's columns [0, J0) (the rows of the L computed so
//     far: keeps W the inverse of the current L), then the solve and update
//     restricted to columns [0, J0 + 128) (W stays unit lower triangular),
//     n^3 / 3 flops in all.
struct LuFold {
  const int* w;      // W slots
  const int* lw;     // (l, W) copy pairs (unused when tri)
  const int* fw;     // (F, W) pairs (triangular solve)
  const int* fwww;   // (F, W, W, W) quads (update GEMM)
  cudaEvent_t ev_l;  // external event gating l (nullptr: resident)
  bool tri;          // W = L^-1 (explicit inverse) instead of L^-1 P l
  // Schur nodes, optional: C = rt U^-1 in slot G as well — G <- rt, then per
  // outer block J (once U's block row J is final) C_J = G_J U_JJ^-1 (right
  // solve) and G[:, J0 + 128:] -= C_J U[J, J0 + 128:].  Leaves only
  // out = r - C W after the factorization.
  const int* gf = nullptr;     // (G, F) pairs (nullptr: no C fold)
  const int* gfgg = nullptr;   // (G, F, G, G) quads
  const int* rtg = nullptr;    // (rt, G) copy pairs
  cudaEvent_t ev_rtr = nullptr;
};

// variant_count (default: count) picks the blocking variant (panel extension into
// the next block, GEMM caps) — the variants round differently, so a DAG level
// keeps the variant of its NODE count even when its distinct pivots are few
// (bri_level_batch): results then do not depend on how much work is shared.
int getrf_device(bri_arena* ar, cudaStream_t s, const int* dev_slots, const int* dev_ffff, const int* dev_ff,
                 int count, const LuLayout& L, const LuScratch& sc, const LuFold* fold = nullptr,
                 int variant_count = -1) {
  const int vcount = variant_count >= 0 ? variant_count : count;
  const ArenaView& v = ar->v;
  const int n = v.n;
  bri_ctx* ctx = ar->ctx;
  cudaStream_t s1 = ctx->side;
  BRI_CHECK(launch_pi_init(sc.pi, n, count, sc.scale_bits, sc.pairs, L.pair_stride, s));
  BRI_CHECK(launch_maxabs(v, dev_slots, count, sc.scale_bits, s));
  const int nbi = panel_width(n);
  const int outer = LU_OUTER;
  const size_t per = (size_t)((n + TRSM_BLOCK - 1) / TRSM_BLOCK) * TRSM_BLOCK * TRSM_BLOCK;
  if (int rc = ctx->dinv.ensure(2 * per * count * sizeof(double), s)) return rc;
  double* dl = static_cast<double*>(ctx->dinv.ptr);

  // factor the outer block [J0, J0 + W) whose columns are up to date (stream s),
  // carrying every inner panel's interchanges / solve / update on to columns
  // [J0 + W, cext) as well; `ext_ready`: event to wait on before the first of
  // those touches [J0 + W, cext) (nullptr: already up to date)
  // ext_ready, split (default; BRI_EXT_SPLIT=0 restores the wait): the chain does not wait for
  // the side stream's update of [J0 + W, cext) before the block's first row panel (the CUPTI
  // timeline of config 2 showed ~29 us of stall there per outer block, 3.8 ms per step) — the
  // first inner panel handles the block's own columns at once, and its carry-over to the
  // extension columns runs on a third stream once they are up to date, overlapping the second
  // inner panel, whose row panel is the first to touch them on the chain.  Same arithmetic per
  // element either way.
  static const bool ext_split = [] {
    const char* e = getenv("BRI_EXT_SPLIT");
    return e == nullptr || e[0] != '0';
  }();
  // few factorizations in flight: the chain kernels trigger their dependents early (pdl_trigger)
  static const bool early_env = [] {
    const char* e = getenv("BRI_PDL_EARLY");
    return e == nullptr || e[0] != '0';
  }();
  const bool early = early_env && bri::pdl_enabled() && vcount <= 2;
  auto factor_block = [&](int J0, int W, int pidx, int cext, cudaEvent_t ext_ready) -> int {
    bool pending_y = false;
    for (int j0 = J0; j0 < J0 + W; j0 += nbi, ++pidx) {
      const int w = (J0 + W - j0) < nbi ? (J0 + W - j0) : nbi;
      BRI_CHECK(launch_panel(v, dev_slots, count, j0, w, pidx, sc, n, L.pair_stride, s, early));
      const bool split = ext_split && j0 == J0 && ext_ready != nullptr && cext > J0 + W && n - j0 - w > 0;
      if (split) {
        cudaStream_t s3 = ctx->side3;
        BRI_CHECK(cudaEventRecord(ctx->ev_p, s));
        BRI_CHECK(launch_rowpanel(v, dev_slots, count, j0, w, pidx, J0, J0 + W, sc, n, L.pair_stride, s, true, early));
        const int right_in = J0 + W - j0 - w;
        if (right_in > 0)
          if (int rc = gemm_call(ar, s, dev_ffff, count, n - j0 - w, right_in, w, j0 + w, j0, j0, j0 + w, j0 + w,
                                 j0 + w, -1.0, 1.0, 0, 0, early))
            return rc;
        BRI_CHECK(cudaStreamWaitEvent(s3, ctx->ev_p, 0));
        BRI_CHECK(cudaStreamWaitEvent(s3, ext_ready, 0));
        BRI_CHECK(launch_rowpanel(v, dev_slots, count, j0, w, pidx, J0 + W, cext, sc, n, L.pair_stride, s3, false));
        if (int rc = gemm_call(ar, s3, dev_ffff, count, n - j0 - w, cext - (J0 + W), w, j0 + w, j0, j0, J0 + W,
                               j0 + w, J0 + W, -1.0, 1.0))
          return rc;
        BRI_CHECK(cudaEventRecord(ctx->ev_y, s3));
        pending_y = true;
        continue;
      }
      if (j0 == J0 && ext_ready) BRI_CHECK(cudaStreamWaitEvent(s, ext_ready, 0));
      if (pending_y) {
        BRI_CHECK(cudaStreamWaitEvent(s, ctx->ev_y, 0));
        pending_y = false;
      }
      BRI_CHECK(launch_rowpanel(v, dev_slots, count, j0, w, pidx, J0, cext, sc, n, L.pair_stride, s, true, early));
      const int right = cext - j0 - w;
      if (right > 0 && n - j0 - w > 0) {
        if (int rc = gemm_call(ar, s, dev_ffff, count, n - j0 - w, right, w, j0 + w, j0, j0, j0 + w, j0 + w,
                               j0 + w, -1.0, 1.0, 0, 0, early))
          return rc;
      }
    }
    if (pending_y) BRI_CHECK(cudaStreamWaitEvent(s, ctx->ev_y, 0));
    return 0;
  };
  // apply block J's interchanges / U12 solve / rank-W update to columns [c0, c1)
  // (cap > 0: the GEMM runs persistent on at most `cap` CTAs, leaving SMs to
  // the critical path that factors the next block concurrently)
  auto update_cols = [&](cudaStream_t st, int J0, int W, int pidx0, int c0, int c1, int cap) -> int {
    if (c1 <= c0) return 0;
    BRI_CHECK(launch_trsm_fused(ar->tmA, ar->tmB32, ar->tmB16, v, dev_ff, count, dl, true, J0, W, c0, c1 - c0, false, st));
    return gemm_call(ar, st, dev_ffff, count, n - J0 - W, c1 - c0, W, J0 + W, J0, J0, c0, J0 + W, c0, -1.0, 1.0,
                     cap);
  };
  // Few factorizations in flight: their panel chain is the critical path and
  // would otherwise wait for the trailing GEMM's CTAs to drain (measured on
  // config 2: cap 80 -> 37.0 ms/step vs 39.4 uncapped).  Large batches keep
  // every SM busy with panels of their own, so their updates run uncapped.
  static const int trail_cap_env = [] {
    const char* e = getenv("BRI_TRAIL_CAP");
    return e ? atoi(e) : -1;
  }();
  const int trail_cap = trail_cap_env >= 0 ? trail_cap_env : (vcount <= 2 ? 80 : 0);

  static const int fold_cap_env = [] {
    const char* e = getenv("BRI_FOLD_CAP");
    return e ? atoi(e) : -1;
  }();
  const int fold_cap = fold_cap_env >= 0 ? fold_cap_env : (vcount <= 2 ? 48 : 0);
  // The caps pay while the pivot chain is the critical path (n <= 4096); for
  // larger orders the bulk updates are, and every SM should take them:
  // measured on one node + inversion (tools/sweep_caps_large.sh), uncapped vs
  // capped: b = 8192 193.5 -> 166.4 ms, b = 20480 2685 -> 2242 ms; per-block
  // capping once n - J0 <= 4096 (BRI_CAP_ROWS=4096) measured 170 / 2277 ms.
  // (Round 1 saw wrong config-5 blocks with both caps forced on; the cause was
  // the tall-panel pivot race in lu.cu, which long-lived capped GEMMs made
  // likely — fixed, and with both caps forced config 5 now returns the
  // uncapped run's exact bits.  The n <= 4096 limit is a speed choice.)
  static const int cap_rows_env = [] {
    const char* e = getenv("BRI_CAP_ROWS");
    return e ? atoi(e) : -1;
  }();
  const int cap_rows = cap_rows_env >= 0 ? cap_rows_env : (n > 4096 ? 0 : 0x7fffffff);
  // Default caps follow the work: the trailing update of block J shrinks like (n - J0)^2, the
  // fold like (n - J0) * n, and the fold has no deadline but the end of the factorization, so it
  // gets the SMs the trailing update (which the chain waits for, one block behind) no longer
  // needs to finish inside one block of the chain (~190 us at ~0.16 TFLOP/s per CTA on K = 128
  // tiles): trail(J) = 132 r^2 clamped to [24, 80], fold(J) = 124 - trail(J + 2) — the fold runs
  // about two blocks behind the chain — with r = (n - J0) / n; the chain keeps 16 SMs for its two
  // resident panel clusters.  With the fixed 80 / 48 pair the fold trailed the chain by ~8 blocks
  // on config 2 and finished 1.3 ms after it on 48 SMs (CUPTI timeline); giving the trailing
  // update 100 CTAs early on starved the fold instead (24 CTAs: 1 ms per block).
  // BRI_DYN_CAPS=0 or an explicit BRI_TRAIL_CAP / BRI_FOLD_CAP keeps fixed caps.
  static const bool dyn_caps_env = [] {
    const char* e = getenv("BRI_DYN_CAPS");
    return e == nullptr || e[0] != '0';
  }();
  const bool dyn_caps = dyn_caps_env && trail_cap_env < 0 && fold_cap_env < 0 && vcount <= 2;
  auto capped = [&](int J0, int cap, bool trailing) {
    if ((n - J0) > cap_rows || cap <= 0) return 0;
    if (!dyn_caps) return cap;
    static const int cap_a = env_or("BRI_CAP_A", 132), cap_hi = env_or("BRI_CAP_HI", 80),
                     cap_lag = env_or("BRI_CAP_LAG", 2);
    auto trail_at = [&](int j0) {
      const double r = j0 < n ? (double)(n - j0) / n : 0.0;
      const int t = (int)(cap_a * r * r + 0.5);
      return t < 24 ? 24 : (t > cap_hi ? cap_hi : t);
    };
    return trailing ? trail_at(J0) : 124 - trail_at(J0 + cap_lag * outer);
  };
  // W <- L11^-1 P_J W on block J's rows, then W[N0:, :] -= L21 W[J rows, :]
  auto fold_block = [&](cudaStream_t st, int J0, int W, int pidx0, int npan) -> int {
    const bool tri = fold->tri;
    const int ncol = tri ? J0 + W : n;
    if (J0 == 0) {
      if (tri) {
        BRI_CHECK(launch_identity(v, fold->w, 1, count, st));
      } else {
        if (fold->ev_l) BRI_CHECK(cudaStreamWaitEvent(st, fold->ev_l, cudaEventWaitExternal));
        BRI_CHECK(launch_copy(v, fold->lw, count, st));
      }
    }
    BRI_CHECK(launch_laswp(v, fold->w, count, J0, W, nbi, pidx0, npan, 0, tri ? J0 : n, 0, 0, sc, n,
                           L.pair_stride, st));
    BRI_CHECK(launch_trsm_fused(ar->tmA, ar->tmB32, ar->tmB16, v, fold->fw, count, dl, true, J0, W, 0, ncol, tri, st));
    if (n - J0 - W > 0)
      return gemm_call(ar, st, fold->fwww, count, n - J0 - W, ncol, W, J0 + W, J0, J0, 0, J0 + W, 0, -1.0, 1.0,
                       capped(J0, fold_cap, false));
    return 0;
  };
  double* du = dl + per * count;
  auto fold_c = [&](cudaStream_t st, int J0, int W) -> int {
    if (!fold || !fold->gf) return 0;
    if (J0 == 0) {
      if (fold->ev_rtr) BRI_CHECK(cudaStreamWaitEvent(st, fold->ev_rtr, cudaEventWaitExternal));
      BRI_CHECK(launch_copy(v, fold->rtg, count, st));
    }
    BRI_CHECK(launch_dinv(v, dev_slots, count, false, du, J0 / TRSM_BLOCK, (W + TRSM_BLOCK - 1) / TRSM_BLOCK, st));
    BRI_CHECK(launch_rtrsm(v, fold->gf, count, du, J0, W, st));
    if (n - J0 - W > 0)
      return gemm_call(ar, st, fold->gfgg, count, n, n - J0 - W, W, 0, J0, J0, J0 + W, 0, J0 + W, -1.0, 1.0,
                       capped(J0, fold_cap, false));
    return 0;
  };
  // C part of block J once its U row block is final (recorded as ev_b on s1)
  auto fold_c_after_b = [&](int J0, int W) -> int {
    if (!fold || !fold->gf) return 0;
    BRI_CHECK(cudaStreamWaitEvent(ctx->side2, ctx->ev_b, 0));
    return fold_c(ctx->side2, J0, W);
  };
  // hand block J (factored, its L11 inverse in dl, both ordered before `ev`
  // on `from`) to the fold stream
  cudaStream_t s2 = ctx->side2;
  auto fold_after = [&](cudaStream_t from, int J0, int W, int pidx0, int npan) -> int {
    if (!fold) return 0;
    BRI_CHECK(cudaEventRecord(ctx->ev_d, from));
    BRI_CHECK(cudaStreamWaitEvent(s2, ctx->ev_d, 0));
    return fold_block(s2, J0, W, pidx0, npan);
  };
  // Left-side interchanges (L columns of earlier blocks): applied per block (left = 1), skipped
  // (the folded path never reads L, left = 0), or deferred — large batches snapshot pi after
  // each block and reorder every L column once at the end (laswp_deferred; config 3 spent ~2%
  // of its step in the per-block left passes).  Same values either way: only row order moves.
  static const int defer_env = [] {
    const char* e = getenv("BRI_DEFER_LASWP");
    return e ? atoi(e) : 1;
  }();
  const bool defer_left = !fold && defer_env && vcount > 2 && n <= laswp_deferred_max_n() && n > LU_OUTER;
  const int nob = (n + LU_OUTER - 1) / LU_OUTER;
  const int left = (fold || defer_left) ? 0 : 1;   // 0: skip the interchanges of L left of the block

  const int npan_outer = outer / nbi;
  static const bool lookahead = [] {
    const char* e = getenv("BRI_LOOKAHEAD");
    return e == nullptr || e[0] != '0';
  }();
  // Extending the inner panels into the next block trades rank-128 GEMM work
  // for rank-32 work: a win when the panel chain is the critical path (few
  // factorizations: config 2 32.5 -> 31.4 ms/step), a loss when a large batch
  // keeps every SM busy anyway (config 3 1.52 -> 1.57 s).
  static const int extend_env = [] {
    const char* e = getenv("BRI_LU_EXTEND");
    return e ? atoi(e) : -1;
  }();
  const bool extend = lookahead && (extend_env >= 0 ? extend_env != 0 : vcount <= 2);
  const int W0 = n < outer ? n : outer;
  const int ext0 = extend ? (n < 2 * outer ? n : 2 * outer) : W0;
  if (int rc = factor_block(0, W0, 0, ext0, nullptr)) return rc;
  for (int J0 = 0, pidx0 = 0; J0 < n; J0 += outer, pidx0 += npan_outer) {
    // block J's panels are done on s (its row permutation is final for rows < J0 + W)
    if (defer_left && J0 + outer < n)
      BRI_CHECK(launch_pi_snapshot(sc.pi, sc.snap, n, nob, J0 / outer, count, s));
    const int W = (n - J0) < outer ? (n - J0) : outer;
    const int npan = (W + nbi - 1) / nbi;
    const int N0 = J0 + W;
    const int WN = (n - N0) < outer ? (n - N0) : outer;
    const int N1 = N0 + WN;
    const int WNN = (n - N1) < outer ? (n - N1) : outer;
    if ((J0 % TRSM_BLOCK) != 0) return fail_msg("getrf: outer block not aligned to the TRSM block");
    if (WN > 0 && !lookahead) {
      BRI_CHECK(launch_laswp(v, dev_slots, count, J0, W, nbi, pidx0, npan, 0, J0 * left, N0, n, sc, n,
                             L.pair_stride, s));
      BRI_CHECK(launch_dinv(v, dev_slots, count, true, dl, J0 / TRSM_BLOCK, (W + TRSM_BLOCK - 1) / TRSM_BLOCK, s));
      if (fold)
        if (int rc = fold_block(s, J0, W, pidx0, npan)) return rc;
      if (int rc = update_cols(s, J0, W, pidx0, N0, n, 0)) return rc;
      if (int rc = fold_c(s, J0, W)) return rc;
      if (int rc = factor_block(N0, WN, pidx0 + npan_outer, N1, nullptr)) return rc;
    } else if (WN > 0 && !extend) {
      // critical path: next block's columns, then factor it
      BRI_CHECK(launch_laswp(v, dev_slots, count, J0, W, nbi, pidx0, npan, N0, N1, 0, 0, sc, n,
                             L.pair_stride, s));
      BRI_CHECK(launch_dinv(v, dev_slots, count, true, dl, J0 / TRSM_BLOCK, (W + TRSM_BLOCK - 1) / TRSM_BLOCK, s));
      BRI_CHECK(cudaEventRecord(ctx->ev_a, s));
      if (int rc = fold_after(s, J0, W, pidx0, npan)) return rc;
      if (int rc = update_cols(s, J0, W, pidx0, N0, N1, 0)) return rc;
      // bulk: everything else, concurrently on the side stream
      BRI_CHECK(cudaStreamWaitEvent(s1, ctx->ev_a, 0));
      BRI_CHECK(launch_laswp(v, dev_slots, count, J0, W, nbi, pidx0, npan, 0, J0 * left, N1, n, sc, n,
                             L.pair_stride, s1));
      if (int rc = update_cols(s1, J0, W, pidx0, N1, n, capped(J0, trail_cap, true))) return rc;
      BRI_CHECK(cudaEventRecord(ctx->ev_b, s1));
      if (int rc = fold_c_after_b(J0, W)) return rc;
      if (int rc = factor_block(N0, WN, pidx0 + npan_outer, N1, nullptr)) return rc;
      BRI_CHECK(cudaStreamWaitEvent(s, ctx->ev_b, 0));
    } else if (WN > 0) {
      // block J (and, through its inner panels, block J+1's columns) is done
      BRI_CHECK(cudaEventRecord(ctx->ev_a, s));
      BRI_CHECK(cudaStreamWaitEvent(s1, ctx->ev_a, 0));
      BRI_CHECK(launch_dinv(v, dev_slots, count, true, dl, J0 / TRSM_BLOCK, (W + TRSM_BLOCK - 1) / TRSM_BLOCK, s1));
      if (int rc = fold_after(s1, J0, W, pidx0, npan)) return rc;
      if (WNN > 0) {   // block J+2's columns first: block J+1's inner panels extend into them
        BRI_CHECK(launch_laswp(v, dev_slots, count, J0, W, nbi, pidx0, npan, N1, N1 + WNN, 0, 0, sc, n,
                               L.pair_stride, s1));
        if (int rc = update_cols(s1, J0, W, pidx0, N1, N1 + WNN, 0)) return rc;
        BRI_CHECK(cudaEventRecord(ctx->ev_x, s1));
      }
      BRI_CHECK(launch_laswp(v, dev_slots, count, J0, W, nbi, pidx0, npan, 0, J0 * left, N1 + WNN, n, sc, n,
                             L.pair_stride, s1));
      if (int rc = update_cols(s1, J0, W, pidx0, N1 + WNN, n, capped(J0, trail_cap, true))) return rc;
      BRI_CHECK(cudaEventRecord(ctx->ev_b, s1));
      if (int rc = fold_c_after_b(J0, W)) return rc;
      if (int rc = factor_block(N0, WN, pidx0 + npan_outer, N1 + WNN, WNN > 0 ? ctx->ev_x : nullptr)) return rc;
      BRI_CHECK(cudaStreamWaitEvent(s, ctx->ev_b, 0));
    } else {
      BRI_CHECK(launch_laswp(v, dev_slots, count, J0, W, nbi, pidx0, npan, 0, J0 * left, 0, 0, sc, n,
                             L.pair_stride, s));
      if (fold) {   // last block: its L11 inverse, then W's last rows
        BRI_CHECK(launch_dinv(v, dev_slots, count, true, dl, J0 / TRSM_BLOCK, (W + TRSM_BLOCK - 1) / TRSM_BLOCK, s));
        if (lookahead) {
          if (int rc = fold_after(s, J0, W, pidx0, npan)) return rc;
          if (int rc = fold_c(s2, J0, W)) return rc;
        } else {
          if (int rc = fold_block(s, J0, W, pidx0, npan)) return rc;
          if (int rc = fold_c(s, J0, W)) return rc;
        }
      }
    }
  }
  if (fold && lookahead) {
    BRI_CHECK(cudaEventRecord(ctx->ev_w, s2));
    BRI_CHECK(cudaStreamWaitEvent(s, ctx->ev_w, 0));
  }
  if (defer_left) BRI_CHECK(launch_laswp_deferred(v, dev_slots, count, sc.pi, sc.snap, nob, outer, s));
  BRI_CHECK(launch_diag_check(v, dev_slots, count, sc.scale_bits, sc.status, s));
  return 0;
}

int ensure_dinv(bri_arena* ar, cudaStream_t s, int count) {
  const int n = ar->v.n;
  const size_t per = (size_t)((n + TRSM_BLOCK - 1) / TRSM_BLOCK) * TRSM_BLOCK * TRSM_BLOCK;
  return ar->ctx->dinv.ensure(2 * per * count * sizeof(double), s);
}

// Inverted 64 x 64 diagonal blocks of L and U for `count` factors (ctx->dinv):
// returns pointers to the L and U tables.  after_getrf: the factorization was
// just computed by getrf_device on this stream, which already inverted every
// L diagonal block but those of its last outer block.
int make_dinv(bri_arena* ar, cudaStream_t s, const int* dev_fslots, int count, double** dl, double** du,
              bool after_getrf = false, bool want_l = true) {
  const int n = ar->v.n;
  const size_t per = (size_t)((n + TRSM_BLOCK - 1) / TRSM_BLOCK) * TRSM_BLOCK * TRSM_BLOCK;
  if (int rc = ar->ctx->dinv.ensure(2 * per * count * sizeof(double), s)) return rc;
  *dl = static_cast<double*>(ar->ctx->dinv.ptr);
  *du = *dl + per * count;
  const int l0 = after_getrf ? ((n - 1) / LU_OUTER) * LU_OUTER / TRSM_BLOCK : 0;
  if (want_l) BRI_CHECK(launch_dinv(ar->v, dev_fslots, count, true, *dl, l0, 0, s));
  BRI_CHECK(launch_dinv(ar->v, dev_fslots, count, false, *du, 0, 0, s));
  return 0;
}

// Recursive triangular solve T * W = W on rows [r0, r0 + nr): large GEMMs at
// the top, the fused per-panel solve (trsm.cu) for sub-triangles <= TRSM_LEAF.
// fw: device (F, W) pairs; gemm_fw: device (F, W, W, W) quads.
// tri: (lower only) the right-hand side is unit-lower-triangular — the L sweep of
// an explicit inverse: W[r, c] = 0 for r < c before and after the solve, so
// columns >= r0 + nr are skipped entirely and the leaves start at each
// column's diagonal.
int trsm_rec(bri_arena* ar, cudaStream_t s, const int* fw, const int* gemm_fw, int count, bool lower,
             int r0, int nr, int nrhs, const double* dinv, bool tri = false, int overlap = 0,
             const int* didx = nullptr) {
  const int ncol = tri ? (r0 + nr < nrhs ? r0 + nr : nrhs) : nrhs;
  if (nr <= TRSM_LEAF) {
    BRI_CHECK(launch_trsm_fused(ar->tmA, ar->tmB32, ar->tmB16, ar->v, fw, count, dinv, lower, r0, nr, 0, ncol, tri, s,
                                didx));
    return 0;
  }
  int h = ((nr / 2) + TRSM_BLOCK - 1) / TRSM_BLOCK * TRSM_BLOCK;
  if (h >= nr) h = nr - TRSM_BLOCK;
  if (lower) {
    if (int rc = trsm_rec(ar, s, fw, gemm_fw, count, true, r0, h, nrhs, dinv, tri, overlap, didx)) return rc;
    // W[r0+h : r0+nr, :] -= L[r0+h : r0+nr, r0 : r0+h] * W[r0 : r0+h, :]
    const int gcol = tri ? (r0 + h < nrhs ? r0 + h : nrhs) : nrhs;
    if (int rc = gemm_call(ar, s, gemm_fw, count, nr - h, gcol, h, r0 + h, r0, r0, 0, r0 + h, 0, -1.0, 1.0, 0,
                           overlap))
      return rc;
    return trsm_rec(ar, s, fw, gemm_fw, count, true, r0 + h, nr - h, nrhs, dinv, tri, overlap, didx);
  }
  if (int rc = trsm_rec(ar, s, fw, gemm_fw, count, false, r0 + h, nr - h, nrhs, dinv, false, overlap, didx))
    return rc;
  // W[r0 : r0+h, :] -= U[r0 : r0+h, r0+h : r0+nr] * W[r0+h : r0+nr, :]
  if (int rc = gemm_call(ar, s, gemm_fw, count, h, nrhs, nr - h, r0, r0 + h, r0 + h, 0, r0, 0, -1.0, 1.0, 0,
                         overlap))
    return rc;
  return trsm_rec(ar, s, fw, gemm_fw, count, false, r0, h, nrhs, dinv, false, overlap, didx);
}

// Both sweeps of dgetrs on W (already row-permuted): L then U.
int getrs_sweeps(bri_arena* ar, cudaStream_t s, const int* dev_f, const int* fw, const int* gemm_fw, int count,
                 bool tri_rhs = false, bool after_getrf = false, int overlap = 0) {
  double *dl = nullptr, *du = nullptr;
  if (int rc = make_dinv(ar, s, dev_f, count, &dl, &du, after_getrf)) return rc;
  const int n = ar->v.n;
  if (int rc = trsm_rec(ar, s, fw, gemm_fw, count, true, 0, n, n, dl, tri_rhs, overlap)) return rc;
  return trsm_rec(ar, s, fw, gemm_fw, count, false, 0, n, n, du, false, overlap);
}

// Run a hot-path kernel sequence as a CUDA graph.  The sequence for a given
// key (operation, geometry, batch size, and the device buffers it reads) is
// issued eagerly the first time, captured on the second, and replayed from
// then on: ~1000 dependent launches per b = 4096 node become one graph launch.
// Item arrays and scratch live at fixed device addresses, so new slot lists
// only need a fresh upload before the replay.  Work is ordered after the
// caller's stream `s` and the caller's stream waits for it.
template <class F>
int run_graphed(bri_ctx* ctx, cudaStream_t s, const std::vector<uintptr_t>& key, F&& issue) {
  static const bool enabled = [] {
    const char* e = getenv("BRI_GRAPHS");
    return e == nullptr || e[0] != '0';
  }();
  if (!enabled) return issue(s);
  cudaStream_t g = ctx->gstream;
  BRI_CHECK(cudaEventRecord(ctx->ev_in, s));
  BRI_CHECK(cudaStreamWaitEvent(g, ctx->ev_in, 0));
  int rc = 0;
  GraphEntry* hit = nullptr;
  for (auto& e : ctx->graphs)
    if (e.key == key) hit = &e;
  if (hit != nullptr) {
    BRI_CHECK(cudaGraphLaunch(hit->exec, g));
    bri::g_launches.fetch_add(hit->kernels, std::memory_order_relaxed);
    for (int q = 0; q < FLOP_KINDS; ++q) bri::count_flops(q, (double)hit->flops[q]);
  } else {
    {
      long long f0[FLOP_KINDS];
      for (int q = 0; q < FLOP_KINDS; ++q) f0[q] = bri::tl_flops[q];
      BRI_CHECK(cudaStreamBeginCapture(g, cudaStreamCaptureModeThreadLocal));
      rc = issue(g);
      long long fcap[FLOP_KINDS];
      for (int q = 0; q < FLOP_KINDS; ++q) fcap[q] = bri::tl_flops[q] - f0[q];
      cudaGraph_t graph = nullptr;
      const cudaError_t e = cudaStreamEndCapture(g, &graph);
      if (rc != 0) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
      }
      if (e != cudaSuccess) return fail("cudaStreamEndCapture", e);
      size_t nnodes = 0;
      BRI_CHECK(cudaGraphGetNodes(graph, nullptr, &nnodes));
      std::vector<cudaGraphNode_t> nodes(nnodes);
      long long kernels = 0;
      if (nnodes) {
        BRI_CHECK(cudaGraphGetNodes(graph, nodes.data(), &nnodes));
        for (auto nd : nodes) {
          cudaGraphNodeType ty;
          if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel) ++kernels;
        }
      }
      cudaGraphExec_t exec = nullptr;
      const cudaError_t e2 = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      if (e2 != cudaSuccess) return fail("cudaGraphInstantiate", e2);
      if (ctx->graphs.size() >= 16) {
        cudaGraphExecDestroy(ctx->graphs.front().exec);
        ctx->graphs.erase(ctx->graphs.begin());
      }
      GraphEntry ent{key, exec, kernels, {}};
      for (int q = 0; q < FLOP_KINDS; ++q) ent.flops[q] = fcap[q];
      ctx->graphs.push_back(ent);
      BRI_CHECK(cudaGraphLaunch(exec, g));
      // the captured launches went through count_launch() during capture
    }
  }
  BRI_CHECK(cudaEventRecord(ctx->ev_out, g));
  BRI_CHECK(cudaStreamWaitEvent(s, ctx->ev_out, 0));
  return rc;
}

std::vector<uintptr_t> graph_key(int kind, bri_arena* ar, int count, const void* items) {
  const bri_ctx* c = ar->ctx;
  return {(uintptr_t)kind, (uintptr_t)ar->v.n, (uintptr_t)ar->v.ld, (uintptr_t)ar->v.nslots,
          (uintptr_t)ar->v.base, (uintptr_t)count, (uintptr_t)items, (uintptr_t)c->lu.ptr,
          (uintptr_t)c->dinv.ptr};
}

// ---------------------------------------------------------------- misc kernels
__global__ void axpby_kernel(ArenaView a, const int* items, double alpha, double beta) {
  const int* it = items + 3 * blockIdx.y;
  const double* x = a.base + (long long)it[0] * a.slot_elems;
  const double* y = a.base + (long long)it[1] * a.slot_elems;
  double* o = a.base + (long long)it[2] * a.slot_elems;
  for (int j = blockIdx.x; j < a.n; j += gridDim.x)
    for (int i = threadIdx.x; i < a.n; i += blockDim.x) {
      const long long off = i + (long long)j * a.ld;
      o[off] = alpha * x[off] + beta * y[off];
    }
}

__global__ void transpose_kernel(ArenaView a, const int* items) {
  __shared__ double tile[32][33];
  const int* it = items + 2 * blockIdx.z;
  const double* src = a.base + (long long)it[0] * a.slot_elems;
  double* dst = a.base + (long long)it[1] * a.slot_elems;
  const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = i0 + threadIdx.x, j = j0 + r;
    if (i < a.n && j < a.n) tile[r][threadIdx.x] = src[i + (long long)j * a.ld];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = j0 + threadIdx.x, j = i0 + r;
    if (i < a.n && j < a.n) dst[i + (long long)j * a.ld] = tile[threadIdx.x][r];
  }
}

// dst(i, pi[x]) = src(x, i) in X-world (items: (src, dst) pairs, fidx: factor index of
// each item's permutation): the last step of a right-side solve C = rt p^-1 computed
// as its transpose (C^T = P (L^T)^-1 (U^T)^-1 rt^T) — transpose back and apply P, in one
// pass; reads and writes stay coalesced through a 32 x 32 smem tile.
__global__ void transpose_permute_kernel(ArenaView a, const int* items, const int* pi, int pi_stride,
                                         const int* fidx) {
  __shared__ double tile[32][33];
  const int* it = items + 2 * blockIdx.z;
  const double* src = a.base + (long long)it[0] * a.slot_elems;
  double* dst = a.base + (long long)it[1] * a.slot_elems;
  const int* p = pi + (long long)fidx[blockIdx.z] * pi_stride;
  const int x0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {   // src(x, i): x contiguous for fixed i
    const int x = x0 + threadIdx.x, i = i0 + r;
    if (x < a.n && i < a.n) tile[r][threadIdx.x] = src[x + (long long)i * a.ld];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {   // dst(i, pi[x]): i contiguous for fixed x
    const int i = i0 + threadIdx.x, x = x0 + r;
    if (x < a.n && i < a.n) dst[i + (long long)p[x] * a.ld] = tile[threadIdx.x][r];
  }
}

// Copy row-major blocks M[i*n : (i+1)*n, j*n : (j+1)*n] of a dense row-major
// matrix (leading dim ldm) into arena slots.  items: (block row i, block col j,
// slot), 0-based.  Arena slots hold the row-major block bytes (ld stride).
__global__ void gather_kernel(ArenaView a, const double* M, long long ldm, const int* items) {
  const int* it = items + 3 * blockIdx.y;
  const long long r0 = (long long)it[0] * a.n, c0 = (long long)it[1] * a.n;
  double* dst = a.base + (long long)it[2] * a.slot_elems;
  for (int r = blockIdx.x; r < a.n; r += gridDim.x) {
    const double* src = M + (r0 + r) * ldm + c0;
    double* d = dst + (long long)r * a.ld;
    for (int c = threadIdx.x; c < a.n; c += blockDim.x) d[c] = src[c];
  }
}

// Padded / element-permuted gather: slot (row r, col c) of block (bi, bj) =
// [[M, 0], [0, I]] at element (rmap[bi*n + r], cmap[bj*n + c]) — the shifted
// window views of padded layouts (reference providers.py:203-271, 380-402).
__global__ void gather_elements_kernel(ArenaView a, const double* M, long long ldm, int m, const int* rmap,
                                       const int* cmap, const int* items) {
  const int* it = items + 3 * blockIdx.y;
  const int* rm = rmap + (long long)it[0] * a.n;
  const int* cm = cmap + (long long)it[1] * a.n;
  double* dst = a.base + (long long)it[2] * a.slot_elems;
  for (int r = blockIdx.x; r < a.n; r += gridDim.x) {
    const int R = rm[r];
    double* d = dst + (long long)r * a.ld;
    for (int c = threadIdx.x; c < a.n; c += blockDim.x) {
      const int C = cm[c];
      d[c] = (R < m && C < m) ? M[(long long)R * ldm + C] : ((R >= m && R == C) ? 1.0 : 0.0);
    }
  }
}

__global__ void fp64_peak_kernel(double* sink, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma_8x8x4(c[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5678) sink[0] = s;
}

}  // namespace

// NVTX range per C-ABI hot call (SURVEY §5 tracing): nsys / ncu --nvtx see the
// level structure (schur / level batches, inversions, factorizations) directly.
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
};
#define BRI_NVTX(name) NvtxScope bri_nvtx_scope_(name)

// ==================================================================== C ABI
extern "C" {

int bri_version(void) { return 100; }

long long bri_launch_count(void) { return bri::g_launches.load(std::memory_order_relaxed); }

long long bri_flop_count(int kind) {
  if (kind < 0 || kind >= bri::FLOP_KINDS) return -1;
  return bri::g_flops[kind].load(std::memory_order_relaxed);
}

const char* bri_last_error(void) { return g_last_error.c_str(); }

int bri_ctx_create(int device, bri_ctx** out) {
  if (out == nullptr) return fail_msg("bri_ctx_create: null out");
  BRI_CHECK(cudaSetDevice(device));
  if (get_encoder() == nullptr) return fail_msg("cuTensorMapEncodeTiled unavailable (driver too old?)");
  BRI_CHECK(configure_gemm());
  BRI_CHECK(configure_lu());
  BRI_CHECK(configure_small());
  BRI_CHECK(configure_trsm());
  bri_ctx* c = new bri_ctx();
  c->device = device;
  int prio_low = 0, prio_high = 0;
  BRI_CHECK(cudaDeviceGetStreamPriorityRange(&prio_low, &prio_high));
  // the bulk trailing updates yield to the critical path (panels) when SMs free up
  BRI_CHECK(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, prio_low));
  BRI_CHECK(cudaEventCreateWithFlags(&c->ev_a, cudaEventDisableTiming));
  BRI_CHECK(cudaEventCreateWithFlags(&c->ev_b, cudaEventDisableTiming));
  BRI_CHECK(cudaEventCreateWithFlags(&c->ev_x, cudaEventDisableTiming));
  BRI_CHECK(cudaEventCreateWithFlags(&c->ev_d, cudaEventDisableTiming));
  BRI_CHECK(cudaEventCreateWithFlags(&c->ev_w, cudaEventDisableTiming));
  BRI_CHECK(cudaStreamCreateWithPriority(&c->side2, cudaStreamNonBlocking, prio_low));
  BRI_CHECK(cudaStreamCreateWithPriority(&c->side3, cudaStreamNonBlocking, prio_high));
  BRI_CHECK(cudaEventCreateWithFlags(&c->ev_p, cudaEventDisableTiming));
  BRI_CHECK(cudaEventCreateWithFlags(&c->ev_y, cudaEventDisableTiming));
  BRI_CHECK(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
  BRI_CHECK(cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming));
  BRI_CHECK(cudaStreamCreateWithPriority(&c->gstream, cudaStreamNonBlocking, prio_high));
  *out = c;
  return 0;
}

void bri_ctx_destroy(bri_ctx* ctx) {
  if (ctx == nullptr) return;
  cudaDeviceSynchronize();
  if (ctx->items.ptr) cudaFree(ctx->items.ptr);
  if (ctx->lu.ptr) cudaFree(ctx->lu.ptr);
  if (ctx->dinv.ptr) cudaFree(ctx->dinv.ptr);
  for (auto& g : ctx->graphs) cudaGraphExecDestroy(g.exec);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->gstream) cudaStreamDestroy(ctx->gstream);
  if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
  if (ctx->ev_out) cudaEventDestroy(ctx->ev_out);
  if (ctx->ev_a) cudaEventDestroy(ctx->ev_a);
  if (ctx->ev_b) cudaEventDestroy(ctx->ev_b);
  if (ctx->ev_x) cudaEventDestroy(ctx->ev_x);
  if (ctx->ev_d) cudaEventDestroy(ctx->ev_d);
  if (ctx->ev_w) cudaEventDestroy(ctx->ev_w);
  if (ctx->side2) cudaStreamDestroy(ctx->side2);
  if (ctx->ev_p) cudaEventDestroy(ctx->ev_p);
  if (ctx->ev_y) cudaEventDestroy(ctx->ev_y);
  if (ctx->side3) cudaStreamDestroy(ctx->side3);
  for (int k = 0; k < bri_ctx::NSTAGE; ++k) {
    if (ctx->stage[k]) cudaFreeHost(ctx->stage[k]);
    if (ctx->stage_ev[k]) cudaEventDestroy(ctx->stage_ev[k]);
  }
  delete ctx;
}

int bri_arena_create(bri_ctx* ctx, double* base, int n, int ld, int nslots, bri_arena** out) {
  if (ctx == nullptr || base == nullptr || out == nullptr) return fail_msg("bri_arena_create: null argument");
  if (n < 1 || ld < n || (ld % 8) != 0 || nslots < 1)
    return fail_msg("bri_arena_create: need n >= 1, ld >= n, ld % 8 == 0, nslots >= 1");
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) return fail_msg("bri_arena_create: base not 16-byte aligned");
  bri_arena* a = new bri_arena();
  a->ctx = ctx;
  a->v.base = base;
  a->v.n = n;
  a->v.ld = ld;
  a->v.slot_elems = (long long)n * ld;
  a->v.nslots = nslots;
  EncodeTiledFn enc = get_encoder();
  const cuuint64_t dims[3] = {(cuuint64_t)ld, (cuuint64_t)n, (cuuint64_t)nslots};
  const cuuint64_t strides[2] = {(cuuint64_t)ld * 8, (cuuint64_t)a->v.slot_elems * 8};
  const cuuint32_t estr[3] = {1, 1, 1};
#if BRI_WIDE_A
  const cuuint32_t boxA[3] = {16, 16, 1};
  const CUtensorMapSwizzle swA = CU_TENSOR_MAP_SWIZZLE_128B;
#else
  const cuuint32_t boxA[3] = {8, 16, 1};
  const CUtensorMapSwizzle swA = CU_TENSOR_MAP_SWIZZLE_64B;
#endif
  const cuuint32_t boxB[3] = {16, 128, 1};
  const cuuint32_t boxB32[3] = {16, 32, 1};
  const cuuint32_t boxB16[3] = {16, 16, 1};
  CUresult r1 = enc(&a->tmA, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, boxA, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swA,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&a->tmB, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, boxB, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r3 = enc(&a->tmB32, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, boxB32, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r4 = enc(&a->tmB16, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, boxB16, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS || r3 != CUDA_SUCCESS || r4 != CUDA_SUCCESS) {
    delete a;
    return fail_msg("cuTensorMapEncodeTiled failed: " + std::to_string((int)r1) + "/" + std::to_string((int)r2));
  }
  *out = a;
  return 0;
}

void bri_arena_destroy(bri_arena* arena) { delete arena; }

int bri_gemm(bri_arena* ar, void* stream, int count, const int* items, int M, int N, int K, int a_r0,
             int a_c0, int b_r0, int b_c0, int c_r0, int c_c0, double alpha, double beta) {
  BRI_NVTX("bri_gemm");
  if (ar == nullptr || items == nullptr || count < 0) return fail_msg("bri_gemm: bad arguments");
  if (((a_r0 | b_r0) & 1) != 0)
    return fail_msg("bri_gemm: a_r0 and b_r0 must be even (TMA boxes start on 16-byte boundaries)");
  if (count == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<int> h(items, items + 4 * count);
  int* dev = nullptr;
  if (int rc = upload(ar->ctx, s, h, &dev)) return rc;
  return gemm_call(ar, s, dev, count, M, N, K, a_r0, a_c0, b_r0, b_c0, c_r0, c_c0, alpha, beta, 0, 1);
}

int bri_axpby(bri_arena* ar, void* stream, int count, const int* items, double alpha, double beta) {
  if (ar == nullptr || items == nullptr || count < 0) return fail_msg("bri_axpby: bad arguments");
  if (count == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<int> h(items, items + 3 * count);
  int* dev = nullptr;
  if (int rc = upload(ar->ctx, s, h, &dev)) return rc;
  const int gx = ar->v.n < 512 ? ar->v.n : 512;
  bri::count_launch();
  axpby_kernel<<<dim3(gx, count), 256, 0, s>>>(ar->v, dev, alpha, beta);
  BRI_CHECK(cudaGetLastError());
  return 0;
}

int bri_transpose(bri_arena* ar, void* stream, int count, const int* items) {
  if (ar == nullptr || items == nullptr || count < 0) return fail_msg("bri_transpose: bad arguments");
  if (count == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<int> h(items, items + 2 * count);
  int* dev = nullptr;
  if (int rc = upload(ar->ctx, s, h, &dev)) return rc;
  const int t = (ar->v.n + 31) / 32;
  bri::count_launch();
  transpose_kernel<<<dim3(t, t, count), dim3(32, 8), 0, s>>>(ar->v, dev);
  BRI_CHECK(cudaGetLastError());
  return 0;
}

int bri_getrf_batch(bri_arena* ar, void* stream, int count, const int* slots, int* ipiv, int* perm,
                    int* status) {
  BRI_NVTX("bri_getrf_batch");
  if (ar == nullptr || slots == nullptr || count < 0) return fail_msg("bri_getrf_batch: bad arguments");
  if (count == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int n = ar->v.n;
  std::vector<int> h(7 * (size_t)count);
  for (int i = 0; i < count; ++i) {
    h[i] = slots[i];
    for (int q = 0; q < 4; ++q) h[count + 4 * i + q] = slots[i];
    h[5 * count + 2 * i] = h[5 * count + 2 * i + 1] = slots[i];
  }
  int* dev = nullptr;
  if (int rc = upload(ar->ctx, s, h, &dev)) return rc;
  LuLayout L = lu_layout(n, count);
  if (int rc = ar->ctx->lu.ensure(L.total, s)) return rc;
  LuScratch sc = lu_scratch(ar->ctx->lu.ptr, L);
  if (int rc = getrf_device(ar, s, dev, dev + count, dev + 5 * count, count, L, sc)) return rc;
  if (ipiv) BRI_CHECK(cudaMemcpyAsync(ipiv, sc.ipiv, (size_t)count * n * 4, cudaMemcpyDeviceToDevice, s));
  if (perm) BRI_CHECK(cudaMemcpyAsync(perm, sc.pi, (size_t)count * n * 4, cudaMemcpyDeviceToDevice, s));
  if (status) BRI_CHECK(cudaMemcpyAsync(status, sc.status, (size_t)count * 4, cudaMemcpyDeviceToDevice, s));
  return 0;
}

int bri_getrs_batch(bri_arena* ar, void* stream, int count, const int* items, const int* perm) {
  BRI_NVTX("bri_getrs_batch");
  if (ar == nullptr || items == nullptr || perm == nullptr || count < 0)
    return fail_msg("bri_getrs_batch: bad arguments");
  if (count == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int n = ar->v.n;
  // layout: [(src,dst) | (F,dst) | (F,dst,dst,dst) | F]
  std::vector<int> h;
  h.reserve(9 * (size_t)count);
  for (int i = 0; i < count; ++i) { h.push_back(items[3 * i + 1]); h.push_back(items[3 * i + 2]); }
  for (int i = 0; i < count; ++i) { h.push_back(items[3 * i]); h.push_back(items[3 * i + 2]); }
  for (int i = 0; i < count; ++i) {
    h.push_back(items[3 * i]);
    for (int q = 0; q < 3; ++q) h.push_back(items[3 * i + 2]);
  }
  for (int i = 0; i < count; ++i) h.push_back(items[3 * i]);
  int* dev = nullptr;
  if (int rc = upload(ar->ctx, s, h, &dev)) return rc;
  BRI_CHECK(launch_permcopy(ar->v, dev, count, perm, n, false, s));
  return getrs_sweeps(ar, s, dev + 8 * count, dev + 2 * count, dev + 4 * count, count);
}

int bri_invert_batch(bri_arena* ar, void* stream, int count, const int* items, int* status) {
  BRI_NVTX("bri_invert_batch");
  if (ar == nullptr || items == nullptr || count < 0) return fail_msg("bri_invert_batch: bad arguments");
  if (count == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int n = ar->v.n;
  if (n <= SMALL_MAX) {
    std::vector<int> h(5 * (size_t)count);
    for (int i = 0; i < count; ++i) {
      h[5 * i + 0] = items[3 * i];
      h[5 * i + 1] = items[3 * i];
      h[5 * i + 2] = items[3 * i];
      h[5 * i + 3] = items[3 * i];
      h[5 * i + 4] = items[3 * i + 2];
    }
    int* dev = nullptr;
    if (int rc = upload(ar->ctx, s, h, &dev)) return rc;
    BRI_CHECK(launch_small_node(ar->v, dev, count, 1, status, s));
    return 0;
  }
  // layout: [F slots | (in,F) pairs | (F,F,F,F) | (F,out) | (F,out,out,out) | (F,F) | (out,F) | out]
  std::vector<int> h;
  h.reserve(18 * (size_t)count);
  for (int i = 0; i < count; ++i) h.push_back(items[3 * i + 1]);
  for (int i = 0; i < count; ++i) { h.push_back(items[3 * i]); h.push_back(items[3 * i + 1]); }
  for (int i = 0; i < count; ++i) for (int q = 0; q < 4; ++q) h.push_back(items[3 * i + 1]);
  for (int i = 0; i < count; ++i) { h.push_back(items[3 * i + 1]); h.push_back(items[3 * i + 2]); }
  for (int i = 0; i < count; ++i) {
    h.push_back(items[3 * i + 1]);
    for (int q = 0; q < 3; ++q) h.push_back(items[3 * i + 2]);
  }
  for (int i = 0; i < count; ++i) { h.push_back(items[3 * i + 1]); h.push_back(items[3 * i + 1]); }
  for (int i = 0; i < count; ++i) { h.push_back(items[3 * i + 2]); h.push_back(items[3 * i + 1]); }
  for (int i = 0; i < count; ++i) h.push_back(items[3 * i + 2]);
  int* dev = nullptr;
  if (int rc = upload(ar->ctx, s, h, &dev)) return rc;
  const int* d_ff = dev + 13 * count;
  const int* d_of = dev + 15 * count;
  const int* d_f = dev;
  const int* d_inf = dev + count;
  const int* d_ffff = dev + 3 * count;
  const int* d_fo = dev + 7 * count;
  const int* d_fooo = dev + 9 * count;
  LuLayout L = lu_layout(n, count);
  if (int rc = ar->ctx->lu.ensure(L.total, s)) return rc;
  if (int rc = ensure_dinv(ar, s, count)) return rc;
  LuScratch sc = lu_scratch(ar->ctx->lu.ptr, L);
  static const int fold_env = [] {
    const char* e = getenv("BRI_FOLD");
    return e ? atoi(e) : -1;
  }();
  const bool fold_on = fold_env >= 0 ? fold_env != 0 : count <= 2;
  auto issue = [&](cudaStream_t st) -> int {
    BRI_CHECK(launch_copy(ar->v, d_inf, count, st));
    if (fold_on) {   // T = L^-1 built during the factorization, then the U sweep
      const LuFold fold{dev + 17 * count, nullptr, d_fo, d_fooo, nullptr, true};
      if (int rc = getrf_device(ar, st, d_f, d_ffff, d_ff, count, L, sc, &fold)) return rc;
      double *dl = nullptr, *du = nullptr;
      if (int rc = make_dinv(ar, st, d_f, count, &dl, &du, true, false)) return rc;
      if (int rc = trsm_rec(ar, st, d_fo, d_fooo, count, false, 0, n, n, du)) return rc;
      BRI_CHECK(launch_colscatter(ar->v, d_of, count, sc.pi, n, st));
      BRI_CHECK(launch_copy(ar->v, d_fo, count, st));
      return 0;
    }
    if (int rc = getrf_device(ar, st, d_f, d_ffff, d_ff, count, L, sc)) return rc;
    // X^-1 = U^-1 L^-1 P (dgetri order): T = U^-1 (L^-1 I) with the L sweep
    // exploiting the triangular identity (n^3/3 instead of n^3), then the
    // column permutation X^-1[:, pi[x]] = T[:, x].  T lives in `out`, the
    // permuted result goes to f (the factors are no longer needed) and back.
    BRI_CHECK(launch_identity(ar->v, d_fo + 1, 2, count, st));
    if (int rc = getrs_sweeps(ar, st, d_f, d_fo, d_fooo, count, true, true)) return rc;
    BRI_CHECK(launch_colscatter(ar->v, d_of, count, sc.pi, n, st));
    BRI_CHECK(launch_copy(ar->v, d_fo, count, st));
    return 0;
  };
  if (int rc = run_graphed(ar->ctx, s, graph_key(1, ar, count, dev), issue)) return rc;
  if (status) BRI_CHECK(cudaMemcpyAsync(status, sc.status, (size_t)count * 4, cudaMemcpyDeviceToDevice, s));
  return 0;
}

int bri_schur_batch_gated(bri_arena* ar, void* stream, int count, const int* items, int* status, void* ev_l,
                          void* ev_rtr);

int bri_schur_batch(bri_arena* ar, void* stream, int count, const int* items, int* status) {
  return bri_schur_batch_gated(ar, stream, count, items, status, nullptr, nullptr);
}

int bri_schur_batch_gated(bri_arena* ar, void* stream, int count, const int* items, int* status, void* ev_l,
                          void* ev_rtr) {
  BRI_NVTX("bri_schur_batch_gated");
  if (ar == nullptr || items == nullptr || count < 0) return fail_msg("bri_schur_batch: bad arguments");
  if (count == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int n = ar->v.n;
  auto I = [&](int i, int k) { return items[7 * i + k]; };  // p, rt, l, r, out, f, w
  if (n <= SMALL_MAX) {
    std::vector<int> h(5 * (size_t)count);
    for (int i = 0; i < count; ++i)
      for (int k = 0; k < 5; ++k) h[5 * i + k] = I(i, k);
    int* dev = nullptr;
    if (int rc = upload(ar->ctx, s, h, &dev)) return rc;
    if (ev_l) BRI_CHECK(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(ev_l), 0));
    if (ev_rtr) BRI_CHECK(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(ev_rtr), 0));
    BRI_CHECK(launch_small_node(ar->v, dev, count, 0, status, s));
    return 0;
  }
  // layout: [F | (p,F) | (F,F,F,F) | (l,W) | (F,W) | (F,W,W,W) | (rt,W,r,out) | (F,F) | W |
  //          (out,F) | (out,F,out,out) | (rt,out) | (out,W,r,F) | (F,out)]   (G = out in the C fold)
  std::vector<int> h;
  h.reserve(36 * (size_t)count);
  for (int i = 0; i < count; ++i) h.push_back(I(i, 5));
  for (int i = 0; i < count; ++i) { h.push_back(I(i, 0)); h.push_back(I(i, 5)); }
  for (int i = 0; i < count; ++i) for (int q = 0; q < 4; ++q) h.push_back(I(i, 5));
  for (int i = 0; i < count; ++i) { h.push_back(I(i, 2)); h.push_back(I(i, 6)); }
  for (int i = 0; i < count; ++i) { h.push_back(I(i, 5)); h.push_back(I(i, 6)); }
  for (int i = 0; i < count; ++i) {
    h.push_back(I(i, 5));
    for (int q = 0; q < 3; ++q) h.push_back(I(i, 6));
  }
  for (int i = 0; i < count; ++i) {
    h.push_back(I(i, 1));
    h.push_back(I(i, 6));
    h.push_back(I(i, 3));
    h.push_back(I(i, 4));
  }
  for (int i = 0; i < count; ++i) { h.push_back(I(i, 5)); h.push_back(I(i, 5)); }
  for (int i = 0; i < count; ++i) h.push_back(I(i, 6));
  for (int i = 0; i < count; ++i) { h.push_back(I(i, 4)); h.push_back(I(i, 5)); }
  for (int i = 0; i < count; ++i) {
    h.push_back(I(i, 4));
    h.push_back(I(i, 5));
    h.push_back(I(i, 4));
    h.push_back(I(i, 4));
  }
  for (int i = 0; i < count; ++i) { h.push_back(I(i, 1)); h.push_back(I(i, 4)); }
  for (int i = 0; i < count; ++i) {
    h.push_back(I(i, 4));
    h.push_back(I(i, 6));
    h.push_back(I(i, 3));
    h.push_back(I(i, 5));
  }
  for (int i = 0; i < count; ++i) { h.push_back(I(i, 5)); h.push_back(I(i, 4)); }
  int* dev = nullptr;
  if (int rc = upload(ar->ctx, s, h, &dev)) return rc;
  const int* d_f = dev;
  const int* d_pf = dev + count;
  const int* d_ffff = dev + 3 * count;
  const int* d_lw = dev + 7 * count;
  const int* d_fw = dev + 9 * count;
  const int* d_fwww = dev + 11 * count;
  const int* d_final = dev + 15 * count;
  LuLayout L = lu_layout(n, count);
  if (int rc = ar->ctx->lu.ensure(L.total, s)) return rc;
  if (int rc = ensure_dinv(ar, s, count)) return rc;
  LuScratch sc = lu_scratch(ar->ctx->lu.ptr, L);
  // the fold pays when the panel chain leaves SMs idle (batches of <= 2:
  // config 2 31.4 -> 30.1 ms/step); large batches are throughput-bound and
  // its rank-128 updates are slower than the recursive sweep (config 3
  // 1.52 -> 1.64 s)
  static const int fold_env = [] {
    const char* e = getenv("BRI_FOLD");
    return e ? atoi(e) : -1;
  }();
  const bool fold_on = fold_env >= 0 ? fold_env != 0 : count <= 2;
  // opt-in: folding C = rt U^-1 as well moves the U sweep into the
  // factorization, but the side streams cannot absorb its 2 n^3 flops next to
  // the panel chain (config 2: 28.5 -> 30.9 ms/step at the best caps, the
  // fold stream ends 4 ms after the last panel)
  static const bool fold_c_on = [] {
    const char* e = getenv("BRI_FOLD_C");
    return e != nullptr && e[0] == '1';
  }();
  auto issue = [&](cudaStream_t s) -> int {
  BRI_CHECK(launch_copy(ar->v, d_pf, count, s));
  // W = P^-1 l  (X-world: W = (p^)^-1 l^ via dgetrs), then out = r - rt * W
  if (fold_on && fold_c_on) {
    // both sweeps folded: W = L^-1 P l and C = rt U^-1 (in `out`) come out of
    // the factorization; F = r - C W, then out <- F
    LuFold fold{dev + 21 * count, d_lw, d_fw, d_fwww, static_cast<cudaEvent_t>(ev_l), false};
    fold.gf = dev + 22 * count;
    fold.gfgg = dev + 24 * count;
    fold.rtg = dev + 28 * count;
    fold.ev_rtr = static_cast<cudaEvent_t>(ev_rtr);
    if (int rc = getrf_device(ar, s, d_f, d_ffff, dev + 19 * count, count, L, sc, &fold)) return rc;
    if (ev_rtr) BRI_CHECK(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(ev_rtr), cudaEventWaitExternal));
    if (int rc = gemm_call(ar, s, dev + 30 * count, count, n, n, n, 0, 0, 0, 0, 0, 0, -1.0, 1.0)) return rc;
    BRI_CHECK(launch_copy(ar->v, dev + 34 * count, count, s));
    return 0;
  }
  if (fold_on) {
    const LuFold fold{dev + 21 * count, d_lw, d_fw, d_fwww, static_cast<cudaEvent_t>(ev_l), false};
    if (int rc = getrf_device(ar, s, d_f, d_ffff, dev + 19 * count, count, L, sc, &fold)) return rc;
    double *dl = nullptr, *du = nullptr;
    if (int rc = make_dinv(ar, s, d_f, count, &dl, &du, true, false)) return rc;
    if (int rc = trsm_rec(ar, s, d_fw, d_fwww, count, false, 0, n, n, du)) return rc;
  } else {
    if (int rc = getrf_device(ar, s, d_f, d_ffff, dev + 19 * count, count, L, sc)) return rc;
    if (ev_l) BRI_CHECK(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(ev_l), cudaEventWaitExternal));
    BRI_CHECK(launch_permcopy(ar->v, d_lw, count, sc.pi, n, false, s));
    if (int rc = getrs_sweeps(ar, s, d_f, d_fw, d_fwww, count, false, true)) return rc;
  }
  if (ev_rtr) BRI_CHECK(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(ev_rtr), cudaEventWaitExternal));
  return gemm_call(ar, s, d_final, count, n, n, n, 0, 0, 0, 0, 0, 0, -1.0, 1.0);
  };
  // gated runs wait on input copies still in flight through external event
  // nodes of the captured graph: the caller records the same (persistent)
  // events before every launch, so the graph keyed on them replays
  std::vector<uintptr_t> key = graph_key(0, ar, count, dev);
  key.push_back((uintptr_t)ev_l);
  key.push_back((uintptr_t)ev_rtr);
  if (int rc = run_graphed(ar->ctx, s, key, issue)) return rc;
  if (status) BRI_CHECK(cudaMemcpyAsync(status, sc.status, (size_t)count * 4, cudaMemcpyDeviceToDevice, s));
  return 0;
}

// One DAG level with its shared work factored out (engine._run_dag): in a level
// of the deduplicated DAG many nodes share their pivot value (config 3: 6,499
// nodes, 2,885 distinct pivots) and many share the pair (pivot, l) and hence
// W = p^-1 l (3,902 distinct).  The reference evaluates each node on its own
// (engine.py:157-180: invert_dense(p), multiply(inv, rt), multiply(l, t));
// here each distinct pivot is factored once, each distinct W solved once, and
// every node only pays its own fused GEMM-subtract.  Same kernels, same
// operand bytes: each W and out is bit-identical to bri_schur_batch's large-
// batch (unfolded) path.
int bri_level_batch_ex(bri_arena* ar, void* stream, int nf, const int* fitems, int ns, const int* sitems,
                       int nt, const int* titems, int nr, const int* ritems, int ng, const int* gitems, int* fstatus,
                       void* ev_l, void* ev_rtr);

int bri_level_batch(bri_arena* ar, void* stream, int nf, const int* fitems, int ns, const int* sitems, int ng,
                    const int* gitems, int* fstatus) {
  return bri_level_batch_ex(ar, stream, nf, fitems, ns, sitems, 0, nullptr, 0, nullptr, ng, gitems, fstatus,
                            nullptr, nullptr);
}

int bri_level_batch_gated(bri_arena* ar, void* stream, int nf, const int* fitems, int ns, const int* sitems,
                          int ng, const int* gitems, int* fstatus, void* ev_l, void* ev_rtr) {
  return bri_level_batch_ex(ar, stream, nf, fitems, ns, sitems, 0, nullptr, 0, nullptr, ng, gitems, fstatus,
                            ev_l, ev_rtr);
}

// ev_l / ev_rtr (optional): the l operands / the rt and r operands are still
// being copied in (first level of a run from pinned host memory); the solves
// wait on ev_l, the GEMM-subtracts on ev_rtr, through external event nodes of
// the captured graph (the caller re-records the same persistent events).
// Right-side solves (nr > 0): for pivots whose nodes share fewer distinct rt than l
// operands, C = rt^ p^-1 is solved once per distinct (pivot, rt) and the nodes compute
// out = r - C * l (the reference's own association, (rt inv(p)) l in X-world) instead of
// out = r - rt * (p^-1 l).  Through transposes, with the left-side kernels:
//   Ft = F^T (per factor, titems (fidx, Ft)): its lower part is U^T (non-unit), upper L^T (unit);
//   S = rt^T;  S <- (U^T)^-1 S;  S <- (L^T)^-1 S;  C(i, pi[x]) = S(x, i)   (C^T = P S)
// ritems: (tidx, rt, S, C), tidx indexing titems.
int bri_level_batch_ex(bri_arena* ar, void* stream, int nf, const int* fitems, int ns, const int* sitems,
                       int nt, const int* titems, int nr, const int* ritems, int ng, const int* gitems, int* fstatus,
                       void* ev_l, void* ev_rtr) {
  BRI_NVTX("bri_level_batch");
  if (ar == nullptr || nf < 0 || ns < 0 || ng < 0 || nt < 0 || nr < 0 || (nf && !fitems) || (ns && !sitems) ||
      (ng && !gitems) || (nt && !titems) || (nr && !ritems))
    return fail_msg("bri_level_batch: bad arguments");
  if (nf == 0 && ns == 0 && ng == 0 && nr == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int n = ar->v.n;
  if (n <= SMALL_MAX) return fail_msg("bri_level_batch: order <= SMALL_MAX uses bri_schur_batch");
  for (int i = 0; i < ns; ++i)
    if (sitems[3 * i] < 0 || sitems[3 * i] >= nf) return fail_msg("bri_level_batch: solve names a bad factor");
  for (int i = 0; i < nt; ++i)
    if (titems[2 * i] < 0 || titems[2 * i] >= nf) return fail_msg("bri_level_batch: transpose names a bad factor");
  for (int i = 0; i < nr; ++i)
    if (ritems[4 * i] < 0 || ritems[4 * i] >= nt) return fail_msg("bri_level_batch: right solve names a bad factor");
  // layout: [F (nf) | (p,F) (nf) | (F,F,F,F) (nf) | (F,F) (nf) | (l,W) (ns) | F_s (ns) | (F_s,W) (ns) |
  //          (F_s,W,W,W) (ns) | fidx (ns) | (rt,W,r,out) (ng)]
  std::vector<int> h;
  h.reserve(9 * (size_t)nf + 10 * (size_t)ns + 4 * (size_t)ng);
  auto F = [&](int f) { return fitems[2 * f + 1]; };
  for (int f = 0; f < nf; ++f) h.push_back(F(f));
  for (int f = 0; f < nf; ++f) { h.push_back(fitems[2 * f]); h.push_back(F(f)); }
  for (int f = 0; f < nf; ++f) for (int q = 0; q < 4; ++q) h.push_back(F(f));
  for (int f = 0; f < nf; ++f) { h.push_back(F(f)); h.push_back(F(f)); }
  for (int i = 0; i < ns; ++i) { h.push_back(sitems[3 * i + 1]); h.push_back(sitems[3 * i + 2]); }
  for (int i = 0; i < ns; ++i) h.push_back(F(sitems[3 * i]));
  for (int i = 0; i < ns; ++i) { h.push_back(F(sitems[3 * i])); h.push_back(sitems[3 * i + 2]); }
  for (int i = 0; i < ns; ++i) {
    h.push_back(F(sitems[3 * i]));
    for (int q = 0; q < 3; ++q) h.push_back(sitems[3 * i + 2]);
  }
  for (int i = 0; i < ns; ++i) h.push_back(sitems[3 * i]);
  for (int g = 0; g < 4 * ng; ++g) h.push_back(gitems[g]);
  // right side: [(F,Ft) (nt) | (rt,S) (nr) | Ft_r (nr) | (Ft_r,S) (nr) | (Ft_r,S,S,S) (nr) | (S,C) (nr) | fidx_r (nr)]
  const size_t r_base = h.size();
  auto Ft = [&](int i) { return titems[2 * ritems[4 * i] + 1]; };
  for (int t = 0; t < nt; ++t) { h.push_back(F(titems[2 * t])); h.push_back(titems[2 * t + 1]); }
  for (int i = 0; i < nr; ++i) { h.push_back(ritems[4 * i + 1]); h.push_back(ritems[4 * i + 2]); }
  for (int i = 0; i < nr; ++i) h.push_back(Ft(i));
  for (int i = 0; i < nr; ++i) { h.push_back(Ft(i)); h.push_back(ritems[4 * i + 2]); }
  for (int i = 0; i < nr; ++i) {
    h.push_back(Ft(i));
    for (int q = 0; q < 3; ++q) h.push_back(ritems[4 * i + 2]);
  }
  for (int i = 0; i < nr; ++i) { h.push_back(ritems[4 * i + 2]); h.push_back(ritems[4 * i + 3]); }
  for (int i = 0; i < nr; ++i) h.push_back(titems[2 * ritems[4 * i]]);
  for (int t = 0; t < nt; ++t) h.push_back(titems[2 * t + 1]);        // Ft slot per transposed factor
  for (int i = 0; i < nr; ++i) h.push_back(ritems[4 * i]);            // its index, per right solve
  int* dev = nullptr;
  if (int rc = upload(ar->ctx, s, h, &dev)) return rc;
  const int* d_tt = dev + r_base;
  const int* d_rs = d_tt + 2 * (size_t)nt;
  const int* d_rft = d_rs + 2 * (size_t)nr;
  const int* d_rfs = d_rft + nr;
  const int* d_rfsss = d_rfs + 2 * (size_t)nr;
  const int* d_rsc = d_rfsss + 4 * (size_t)nr;
  const int* d_rfidx = d_rsc + 2 * (size_t)nr;
  const int* d_tft = d_rfidx + nr;
  const int* d_rtidx = d_tft + nt;
  const int* d_f = dev;
  const int* d_pf = dev + nf;
  const int* d_ffff = dev + 3 * (size_t)nf;
  const int* d_ff = dev + 7 * (size_t)nf;
  const int* d_lw = dev + 9 * (size_t)nf;
  const int* d_fs = d_lw + 2 * (size_t)ns;
  const int* d_fw = d_fs + ns;
  const int* d_fwww = d_fw + 2 * (size_t)ns;
  const int* d_fidx = d_fwww + 4 * (size_t)ns;
  const int* d_g = d_fidx + ns;
  LuLayout L = lu_layout(n, nf > 0 ? nf : 1);
  if (int rc = ar->ctx->lu.ensure(L.total, s)) return rc;
  {
    int most = nf > ns ? nf : ns;
    if (nr > most) most = nr;
    if (int rc = ensure_dinv(ar, s, most)) return rc;
  }
  LuScratch sc = lu_scratch(ar->ctx->lu.ptr, L);
  const size_t per_dinv = (size_t)((n + TRSM_BLOCK - 1) / TRSM_BLOCK) * TRSM_BLOCK * TRSM_BLOCK;
  auto issue = [&](cudaStream_t st) -> int {
    if (nf > 0) {
      BRI_CHECK(launch_copy(ar->v, d_pf, nf, st));
      if (int rc = getrf_device(ar, st, d_f, d_ffff, d_ff, nf, L, sc, nullptr, ng > nf ? ng : nf)) return rc;
    }
    if (ns > 0) {   // W = U^-1 L^-1 P l with the permutation of the solve's factor
      if (ev_l) BRI_CHECK(cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(ev_l), cudaEventWaitExternal));
      BRI_CHECK(launch_permcopy(ar->v, d_lw, ns, sc.pi, n, false, st, d_fidx));
      // diagonal-block inverses once per FACTOR (solves index them through d_fidx); the
      // factorization already inverted L's diagonal blocks but those of its last outer block
      double *dl = nullptr, *du = nullptr;
      if (int rc = make_dinv(ar, st, d_f, nf, &dl, &du, true)) return rc;
      if (int rc = trsm_rec(ar, st, d_fw, d_fwww, ns, true, 0, n, n, dl, false, 1, d_fidx)) return rc;
      if (int rc = trsm_rec(ar, st, d_fw, d_fwww, ns, false, 0, n, n, du, false, 1, d_fidx)) return rc;
    }
    if (nr > 0) {   // C = rt^ p^-1 through the transposed factor (the dinv tables reuse the
                    // region the left-side sweeps used: same stream, strictly after them)
      const int tb = (n + 31) / 32;
      count_launch();
      transpose_kernel<<<dim3(tb, tb, nt), dim3(32, 8), 0, st>>>(ar->v, d_tt);
      BRI_CHECK(cudaGetLastError());
      if (ev_rtr) BRI_CHECK(cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(ev_rtr), cudaEventWaitExternal));
      count_launch();
      transpose_kernel<<<dim3(tb, tb, nr), dim3(32, 8), 0, st>>>(ar->v, d_rs);
      BRI_CHECK(cudaGetLastError());
      double* tl = static_cast<double*>(ar->ctx->dinv.ptr);
      double* tu = tl + per_dinv * nt;
      BRI_CHECK(launch_dinv_t(ar->v, d_tft, nt, true, false, tl, 0, 0, st));    // U^T: lower, non-unit
      BRI_CHECK(launch_dinv_t(ar->v, d_tft, nt, false, true, tu, 0, 0, st));    // L^T: upper, unit
      if (int rc = trsm_rec(ar, st, d_rfs, d_rfsss, nr, true, 0, n, n, tl, false, 0, d_rtidx)) return rc;
      if (int rc = trsm_rec(ar, st, d_rfs, d_rfsss, nr, false, 0, n, n, tu, false, 0, d_rtidx)) return rc;
      count_launch();
      transpose_permute_kernel<<<dim3(tb, tb, nr), dim3(32, 8), 0, st>>>(ar->v, d_rsc, sc.pi, n, d_rfidx);
      BRI_CHECK(cudaGetLastError());
    }
    if (ev_l) BRI_CHECK(cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(ev_l), cudaEventWaitExternal));
    if (ev_rtr) BRI_CHECK(cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(ev_rtr), cudaEventWaitExternal));
    if (ng > 0) return gemm_call(ar, st, d_g, ng, n, n, n, 0, 0, 0, 0, 0, 0, -1.0, 1.0, 0, 1);
    return 0;
  };
  std::vector<uintptr_t> key = graph_key(2, ar, ng, dev);
  key.push_back((uintptr_t)nf);
  key.push_back((uintptr_t)ns);
  key.push_back((uintptr_t)nt);
  key.push_back((uintptr_t)nr);
  key.push_back((uintptr_t)ev_l);
  key.push_back((uintptr_t)ev_rtr);
  if (int rc = run_graphed(ar->ctx, s, key, issue)) return rc;
  if (fstatus && nf > 0)
    BRI_CHECK(cudaMemcpyAsync(fstatus, sc.status, (size_t)nf * 4, cudaMemcpyDeviceToDevice, s));
  return 0;
}

// A whole small-order DAG run (b <= SMALL_MAX) as ONE call and one graph: gather the
// matrix blocks, one one-CTA node launch per level (nodes of a level are independent;
// level l+1 reads level l's outputs), then the final inversions.  All item arrays go to
// the device in one upload; per-level launches inside the graph have no host gaps.
//   gitems: 3 ints (block row, block col, slot), 0-based      -> bri_gather_blocks
//   nitems: 5 ints (p, rt, l, r, out) per node, levels in order; node_status: one int each
//   iitems: 2 ints (in, out) per final inversion; inv_status: one int each (ninv may be 0)
int bri_dag_small(bri_arena* ar, void* stream, const double* M, long long ldm, int ng, const int* gitems,
                  int nlev, const int* lev_counts, const int* nitems, int* node_status, int ninv,
                  const int* iitems, int* inv_status) {
  BRI_NVTX("bri_dag_small");
  if (ar == nullptr || M == nullptr || ng < 0 || nlev < 0 || ninv < 0 || (ng && !gitems) ||
      (nlev && (!lev_counts || !nitems || !node_status)) || (ninv && (!iitems || !inv_status)))
    return fail_msg("bri_dag_small: bad arguments");
  const int n = ar->v.n;
  if (n > SMALL_MAX) return fail_msg("bri_dag_small: order > SMALL_MAX uses the level batches");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int nn = 0;
  for (int l = 0; l < nlev; ++l) {
    if (lev_counts[l] < 0) return fail_msg("bri_dag_small: negative level count");
    nn += lev_counts[l];
  }
  std::vector<int> h;
  h.reserve(3 * (size_t)ng + 5 * (size_t)nn + 5 * (size_t)ninv);
  h.insert(h.end(), gitems, gitems + 3 * (size_t)ng);
  h.insert(h.end(), nitems, nitems + 5 * (size_t)nn);
  for (int i = 0; i < ninv; ++i) {   // the node kernel's inverse mode reads (in, -, -, -, out)
    for (int q = 0; q < 4; ++q) h.push_back(iitems[2 * i]);
    h.push_back(iitems[2 * i + 1]);
  }
  int* dev = nullptr;
  if (int rc = upload(ar->ctx, s, h, &dev)) return rc;
  const int* d_g = dev;
  const int* d_n = dev + 3 * (size_t)ng;
  const int* d_i = d_n + 5 * (size_t)nn;
  std::vector<int> counts(lev_counts, lev_counts + nlev);
  auto issue = [&](cudaStream_t st) -> int {
    if (ng > 0) {
      const int gx = n < 1024 ? n : 1024;
      count_launch();
      gather_kernel<<<dim3(gx, ng), 256, 0, st>>>(ar->v, M, ldm, d_g);
      BRI_CHECK(cudaGetLastError());
    }
    int off = 0;
    for (int l = 0; l < nlev; ++l) {
      BRI_CHECK(launch_small_node(ar->v, d_n + 5 * (size_t)off, counts[l], 0, node_status + off, st));
      off += counts[l];
    }
    if (ninv > 0) BRI_CHECK(launch_small_node(ar->v, d_i, ninv, 1, inv_status, st));
    return 0;
  };
  std::vector<uintptr_t> key = graph_key(5, ar, nn, dev);
  key.push_back((uintptr_t)M);
  key.push_back((uintptr_t)ldm);
  key.push_back((uintptr_t)ng);
  key.push_back((uintptr_t)ninv);
  key.push_back((uintptr_t)node_status);
  key.push_back((uintptr_t)inv_status);
  for (int l = 0; l < nlev; ++l) key.push_back((uintptr_t)counts[l]);
  return run_graphed(ar->ctx, s, key, issue);
}

int bri_gather_blocks(bri_arena* ar, void* stream, const double* M, long long ldm, int count,
                      const int* items) {
  BRI_NVTX("bri_gather_blocks");
  if (ar == nullptr || M == nullptr || items == nullptr || count < 0) return fail_msg("bri_gather_blocks: bad arguments");
  if (count == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<int> h(items, items + 3 * count);
  int* dev = nullptr;
  if (int rc = upload(ar->ctx, s, h, &dev)) return rc;
  const int gx = ar->v.n < 1024 ? ar->v.n : 1024;
  bri::count_launch();
  gather_kernel<<<dim3(gx, count), 256, 0, s>>>(ar->v, M, ldm, dev);
  BRI_CHECK(cudaGetLastError());
  return 0;
}

int bri_gather_elements(bri_arena* ar, void* stream, const double* M, long long ldm, int m, const int* rmap,
                        const int* cmap, int count, const int* items) {
  if (ar == nullptr || M == nullptr || rmap == nullptr || cmap == nullptr || items == nullptr || count < 0)
    return fail_msg("bri_gather_elements: bad arguments");
  if (count == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<int> h(items, items + 3 * count);
  int* dev = nullptr;
  if (int rc = upload(ar->ctx, s, h, &dev)) return rc;
  const int gx = ar->v.n < 1024 ? ar->v.n : 1024;
  bri::count_launch();
  gather_elements_kernel<<<dim3(gx, count), 256, 0, s>>>(ar->v, M, ldm, m, rmap, cmap, dev);
  BRI_CHECK(cudaGetLastError());
  return 0;
}

int bri_store_host(void* stream, double* host, long long ldh, const double* dev, long long ldd, int rows,
                   int cols) {
  if (host == nullptr || dev == nullptr || rows < 0 || cols < 0 || ldh < cols || ldd < cols)
    return fail_msg("bri_store_host: bad arguments");
  if (rows == 0 || cols == 0) return 0;
  BRI_CHECK(cudaMemcpy2DAsync(host, (size_t)ldh * 8, dev, (size_t)ldd * 8, (size_t)cols * 8, rows,
                              cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)));
  return 0;
}

int bri_load_host_blocks(bri_arena* ar, void* stream, const double* host, long long ldh, int count,
                         const int* items) {
  BRI_NVTX("bri_load_host_blocks");
  if (ar == nullptr || host == nullptr || items == nullptr || count < 0 || ldh < ar->v.n)
    return fail_msg("bri_load_host_blocks: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int n = ar->v.n;
  for (int q = 0; q < count; ++q) {
    const int i = items[3 * q], j = items[3 * q + 1], slot = items[3 * q + 2];
    if (i < 0 || j < 0 || slot < 0 || slot >= ar->v.nslots) return fail_msg("bri_load_host_blocks: bad item");
    const double* src = host + (long long)i * n * ldh + (long long)j * n;
    double* dst = ar->v.base + (long long)slot * ar->v.slot_elems;
    BRI_CHECK(cudaMemcpy2DAsync(dst, (size_t)ar->v.ld * 8, src, (size_t)ldh * 8, (size_t)n * 8, (size_t)n,
                                cudaMemcpyHostToDevice, s));
  }
  return 0;
}

int bri_rbf_blocks(bri_arena* ar, void* stream, const double* x, int n, int d, double denom, double ridge,
                   const int* rmap, const int* cmap, int count, const int* items) {
  BRI_NVTX("bri_rbf_blocks");
  if (ar == nullptr || x == nullptr || items == nullptr || n < 1 || d < 1 || count < 0 ||
      (rmap == nullptr) != (cmap == nullptr))
    return fail_msg("bri_rbf_blocks: bad arguments");
  if (count == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<int> h(items, items + 3 * count);
  int* dev = nullptr;
  if (int rc = upload(ar->ctx, s, h, &dev)) return rc;
  const RbfArgs g{x, n, d, denom, ridge, rmap, cmap};
  BRI_CHECK(launch_rbf(g, ar->v.base, ar->v.slot_elems, ar->v.ld, ar->v.n, dev, count, s));
  return 0;
}

int bri_rbf_dense(void* stream, const double* x, int n, int d, double denom, double ridge, double* out,
                  long long ldo) {
  if (x == nullptr || out == nullptr || n < 1 || d < 1 || ldo < (long long)n + 1 || ldo > 0x7fffffffLL)
    return fail_msg("bri_rbf_dense: bad arguments");
  const RbfArgs g{x, n, d, denom, ridge, nullptr, nullptr};
  BRI_CHECK(launch_rbf(g, out, 0, (int)ldo, n + 1, nullptr, 1, static_cast<cudaStream_t>(stream)));
  return 0;
}

int bri_randn_blocks(bri_arena* ar, void* stream, long long m, unsigned long long seed, double shift,
                     const int* rmap, const int* cmap, int count, const int* items) {
  BRI_NVTX("bri_randn_blocks");
  if (ar == nullptr || items == nullptr || m < 1 || count < 0 || (rmap == nullptr) != (cmap == nullptr))
    return fail_msg("bri_randn_blocks: bad arguments");
  if (count == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<int> h(items, items + 3 * count);
  for (int q = 0; q < count; ++q)
    if (h[3 * q] < 0 || h[3 * q + 1] < 0 || h[3 * q + 2] < 0 || h[3 * q + 2] >= ar->v.nslots)
      return fail_msg("bri_randn_blocks: bad item");
  int* dev = nullptr;
  if (int rc = upload(ar->ctx, s, h, &dev)) return rc;
  const RandnArgs g{m, seed, shift, rmap, cmap};
  BRI_CHECK(launch_randn(g, ar->v.base, ar->v.slot_elems, ar->v.ld, ar->v.n, ar->v.n, 0, 0, dev, count, s));
  return 0;
}

int bri_randn_window(void* stream, long long m, unsigned long long seed, double shift, long long row0,
                     long long col0, int rows, int cols, double* out, long long ldo) {
  if (out == nullptr || m < 1 || rows < 1 || cols < 1 || row0 < 0 || col0 < 0 || ldo < cols ||
      ldo > 0x7fffffffLL)
    return fail_msg("bri_randn_window: bad arguments");
  const RandnArgs g{m, seed, shift, nullptr, nullptr};
  BRI_CHECK(launch_randn(g, out, 0, (int)ldo, rows, cols, row0, col0, nullptr, 1, static_cast<cudaStream_t>(stream)));
  return 0;
}

int bri_fp64_peak(void* stream, int iters, double* tflops) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 0;
  BRI_CHECK(cudaGetDevice(&dev));
  BRI_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* sink = nullptr;
  BRI_CHECK(cudaMallocAsync(&sink, 8, s));
  const int blocks = sms * 2, threads = 256;
  cudaEvent_t e0, e1;
  BRI_CHECK(cudaEventCreate(&e0));
  BRI_CHECK(cudaEventCreate(&e1));
  fp64_peak_kernel<<<blocks, threads, 0, s>>>(sink, iters / 4);
  BRI_CHECK(cudaEventRecord(e0, s));
  fp64_peak_kernel<<<blocks, threads, 0, s>>>(sink, iters);
  BRI_CHECK(cudaEventRecord(e1, s));
  BRI_CHECK(cudaEventSynchronize(e1));
  float ms = 0.f;
  BRI_CHECK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  BRI_CHECK(cudaFreeAsync(sink, s));
  const double flops = (double)blocks * (threads / 32) * iters * 8 * (2.0 * 8 * 8 * 4);
  if (tflops) *tflops = flops / (ms * 1e-3) / 1e12;
  return 0;
}

}  // extern "C"
