// Internal (C++) interfaces between the kernel files and the C-ABI layer.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

// A-operand TMA boxes: 16 x 16 doubles with 128-byte swizzle (1) or 8 x 16 with
// 64-byte swizzle (0); the arena's tensor map and dmma_tile.cuh must agree.
#ifndef BRI_WIDE_A
#define BRI_WIDE_A 1
#endif

namespace bri {

// Every kernel launch made by the library bumps this (exported as bri_launch_count).
void count_launch();
enum { FLOP_GEMM = 0, FLOP_TRSM = 1, FLOP_KINDS = 2 };
void count_flops(int kind, double flops);

// Programmatic dependent launch for the LU pivot chain (panel -> row panel ->
// rank-32 update -> next panel, all on one stream): such a kernel is launched
// with cudaLaunchAttributeProgrammaticStreamSerialization so its launch overlaps
// the tail of its predecessor, and it executes griddepcontrol.wait before its
// first global access.  BRI_PDL=0 disables the attribute.
bool pdl_enabled();
inline void pdl_attr(cudaLaunchAttribute& a) {
  a.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a.val.programmaticStreamSerializationAllowed = 1;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Early trigger (`early` launches only: the pivot chain of <= 2 concurrent factorizations): a chain
// kernel lets its dependent become RESIDENT at once — the dependent executes this too before its
// own griddepcontrol.wait, so the residency cascades and the next panel's cluster holds its 8 SMs
// while the current panel still runs.  Without it the panel re-acquires 8 free SMs of one GPC at
// every launch and loses them to the concurrent capped GEMMs (config-2 timeline: stalls of up to
// 270 us with nothing of the chain running).  Memory ordering is unchanged: every dependent still
// waits for its predecessor's completion before touching global memory.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// One-time kernel attribute setup (dynamic shared memory), done at context creation
// so that hot-path sequences can be captured into CUDA graphs on first use.
cudaError_t configure_gemm();
cudaError_t configure_lu();
cudaError_t configure_small();
cudaError_t configure_trsm();

constexpr int NBMAX = 32;        // LU panel width upper bound
constexpr int SMALL_MAX = 96;    // blocks up to this order run the fused one-CTA kernels
constexpr int TRSM_BLOCK = 64;   // diagonal block of the fused triangular solve
#ifndef BRI_TRSM_LEAF
#define BRI_TRSM_LEAF 512
#endif
constexpr int TRSM_LEAF = BRI_TRSM_LEAF;   // recursive solves hand sub-triangles up to this size to trsm.cu
                                           // (256 and 1024 measured no better on configs 2 and 3)
#ifndef BRI_LU_OUTER
#define BRI_LU_OUTER 128
#endif
// outer block width of the two-level LU (multiple of TRSM_BLOCK and NBMAX); 256 measured
// slower on config 2 (33.0 vs 32.4 ms) and equal on config 3
constexpr int LU_OUTER = BRI_LU_OUTER;

// Arena geometry: nslots column-major n x n blocks (X-world), leading dim ld
// (multiple of 8, >= n), slot i at base + i * slot_elems.
struct ArenaView {
  double* base;
  int n;
  int ld;
  long long slot_elems;
  int nslots;
};

struct GemmParams {
  double* base;
  int ld;
  long long slot_elems;
  const int* items;  // device: 4 ints per item (slot A, slot B, slot C_in, slot C_out)
  int M, N, K;
  int a_r0, a_c0, b_r0, b_c0, c_r0, c_c0;
  double alpha, beta;
  int tiles_m, tiles_n;
  int count;      // batch size (set by launch_gemm)
  int max_ctas;   // > 0: persistent launch with at most this many CTAs
  int early;      // 1: skinny launch on the pivot chain triggers its dependent at once (pdl_trigger)
  int overlap;    // 1: persistent launch, one CTA per SM, whose epilogue (straight from the
                  // accumulators) overlaps the next tile's TMA loads; only where nothing runs
                  // concurrently on other streams (it holds every SM until the batch is done)
};

int gemm_smem_bytes();
int skinny_max_k();
long long skinny_max_tiles();
cudaError_t launch_gemm(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmB32,
                        const GemmParams& p, int count, cudaStream_t stream);
cudaError_t launch_scale_copy(const GemmParams& p, int count, cudaStream_t stream);

// ---------------------------------------------------------------- LU pieces
struct LuScratch {
  // device arrays, per item
  int* ipiv;      // n
  int* pi;        // n   (row permutation: (P X)[x] = X[pi[x]])
  int* sigma;     // n   (per panel: source row of each segment position)
  int* pairs;     // npanels * (1 + 2 * NBMAX)
  unsigned long long* scale_bits;  // 1 (max |X| as double bits)
  int* status;    // 1
  int* orig;      // n   (tall panels: original row now at each position)
  int* snap;      // nob * n  (deferred interchanges: inverse of pi after each outer block)
};

// Deferred left-side interchanges of a blocked LU (lu.cu): snapshot pi's inverse after
// outer block J; at the end put every L column of block J into the final row order with
// one gather per column segment (instead of one laswp pass per later block).
cudaError_t launch_pi_snapshot(const int* pi, int* snap, int n, int nob, int J, int count, cudaStream_t s);
cudaError_t launch_laswp_deferred(const ArenaView& a, const int* slots, int count, const int* pi,
                                  const int* snap, int nob, int outer, cudaStream_t s);
int laswp_deferred_max_n();

cudaError_t launch_maxabs(const ArenaView& a, const int* slots, int count,
                          unsigned long long* scale_bits, cudaStream_t s);
cudaError_t launch_copy(const ArenaView& a, const int* pairs, int count, cudaStream_t s);
cudaError_t launch_permcopy(const ArenaView& a, const int* pairs, int count, const int* pi,
                            int pi_stride, bool identity_src, cudaStream_t s, const int* pidx = nullptr);
cudaError_t launch_pi_init(int* pi, int n, int count, unsigned long long* scale_bits, int* pairs, int pair_stride,
                           cudaStream_t s);
// dst X-column pi[x] = src X-column x (column scatter; X-columns are memory rows); pairs (src, dst)
cudaError_t launch_colscatter(const ArenaView& a, const int* pairs, int count, const int* pi, int pi_stride,
                              cudaStream_t s);
cudaError_t launch_identity(const ArenaView& a, const int* slots, int slot_stride, int count, cudaStream_t s);
int panel_width(int n);
int max_panel_rows();  // largest order the register-resident panel factors (16-CTA cluster, 2 rows/thread);
                       // taller panels go through the global-memory tall-panel kernel
cudaError_t launch_panel(const ArenaView& a, const int* slots, int count, int j0, int nb, int pidx,
                         const LuScratch& sc, int n_stride, int pair_stride, cudaStream_t s, bool early = false);
cudaError_t launch_rowpanel(const ArenaView& a, const int* slots, int count, int j0, int nb, int pidx,
                            int cbeg, int cend, const LuScratch& sc, int n_stride, int pair_stride,
                            cudaStream_t s, bool compose_pi = true, bool early = false);
cudaError_t launch_laswp(const ArenaView& a, const int* slots, int count, int J0, int W, int nbi, int pidx0,
                         int npan, int a0, int a1, int b0, int b1, const LuScratch& sc, int n_stride,
                         int pair_stride, cudaStream_t s);
cudaError_t launch_diag_check(const ArenaView& a, const int* slots, int count,
                              const unsigned long long* scale_bits, int* status, cudaStream_t s);

int trsm_smem_bytes();
cudaError_t launch_dinv(const ArenaView& a, const int* fslots, int count, bool lower, double* dinv,
                        int blk0, int nblocks, cudaStream_t s);
// general triangle kind: lower/upper x unit/non-unit diagonal (transposed factors: Uᵀ is
// lower non-unit, Lᵀ upper unit)
cudaError_t launch_dinv_t(const ArenaView& a, const int* fslots, int count, bool lower, bool unit, double* dinv,
                          int blk0, int nblocks, cudaStream_t s);
// X * U[J0:J0+W, J0:J0+W] = B in place on columns [J0, J0 + W) of G, all rows;
// gf: device (G, F) pairs; dinv_u: inverted upper diagonal blocks of F
cudaError_t launch_rtrsm(const ArenaView& a, const int* gf, int count, const double* dinv_u, int J0, int W,
                         cudaStream_t s);
cudaError_t launch_trsm_fused(const CUtensorMap& tmA, const CUtensorMap& tmB32, const CUtensorMap& tmB16,
                              const ArenaView& a, const int* fw, int count, const double* dinv, bool lower, int r0,
                              int nr, int c_off, int nrhs, bool tri_rhs, cudaStream_t s,
                              const int* didx = nullptr);

// Fused one-CTA node / inverse for n <= SMALL_MAX.
// items: 5 ints per item (p, rt, l, r, out); mode 0 = Schur node, 1 = inverse of p.
cudaError_t launch_small_node(const ArenaView& a, const int* items, int count, int mode,
                              int* status, cudaStream_t s);

// LS-SVM kernel system matrix generated on the device (generate.cu).
struct RbfArgs {
  const double* x;  // n x d row-major training inputs (device)
  int n, d;
  double denom;     // -2 sigma^2
  double ridge;     // 1 / gamma
  const int* rmap;  // device view->global maps of length k*bn, or nullptr (identity)
  const int* cmap;
};
// items: (block row, block col, slot) device triples; nullptr = one dense output at base.
cudaError_t launch_rbf(const RbfArgs& g, double* base, long long slot_elems, int ld, int bn, const int* items,
                       int count, cudaStream_t s);

// Seeded Gaussian matrix M = G + shift I generated blockwise on the device (generate.cu).
struct RandnArgs {
  long long m;              // order of M (indices >= m are identity padding)
  unsigned long long seed;  // Philox4x64-10 key word 0
  double shift;             // added to the diagonal
  const int* rmap;          // device view->global maps, or nullptr (identity)
  const int* cmap;
};
// items: (block row, block col, slot) device triples of rows x cols blocks, or
// nullptr = one rows x cols window at (row0, col0) written at base.
cudaError_t launch_randn(const RandnArgs& g, double* base, long long slot_elems, int ld, int rows, int cols,
                         long long row0, long long col0, const int* items, int count, cudaStream_t s);

}  // namespace bri
