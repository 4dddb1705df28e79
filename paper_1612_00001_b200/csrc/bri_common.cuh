// Shared device helpers for the BRI sm_100a kernels: mbarrier / TMA PTX,
// FP64 DMMA (mma.sync f64 -> SASS DMMA.8x8x4), cluster DSMEM access.
//
// Conventions used by every kernel in this library ("X-world"):
//   A row-major b x b block buffer (the reference's C-ordered ndarray,
//   core.py:78-98) is read as its column-major transpose X = A^T, exactly like
//   LAPACK sees `x.data.T` in core.py:249.  Element (i, j) of X lives at
//   base[i + j * ld].  All factorizations / solves / products are written in
//   LAPACK column-major terms on X.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#define BRI_DEVI __device__ __forceinline__

namespace bri {

constexpr double kEps = 2.220446049250313e-16;   // np.finfo(float64).eps
constexpr double kSfmin = 2.2250738585072014e-308;

// ---------------------------------------------------------------- smem ptrs
BRI_DEVI uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
BRI_DEVI void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

BRI_DEVI void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

BRI_DEVI void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

BRI_DEVI void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

BRI_DEVI void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------- TMA
BRI_DEVI void tma_prefetch_desc(const void* desc) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(desc)) : "memory");
}

BRI_DEVI void tma_load_3d(void* smem_dst, const void* desc, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// ---------------------------------------------------------------- DMMA
// D(16x8) += A(16x4) * B(4x8), f64; lane (g = lane>>2, t = lane&3) holds
//   a0 = A[g][t], a1 = A[g+8][t], b0 = B[t][g],
//   c0 = C[g][2t], c1 = C[g][2t+1], c2 = C[g+8][2t], c3 = C[g+8][2t+1].
BRI_DEVI void dmma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// D(8x8) += A(8x4) * B(4x8); a0 = A[g][t], b0 = B[t][g], c0/c1 = C[g][2t..2t+1].
BRI_DEVI void dmma_8x8x4(double (&c)[2], double a0, double b0) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a0), "d"(b0));
}

// ---------------------------------------------------------------- cluster
BRI_DEVI uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

BRI_DEVI uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}

BRI_DEVI void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// Map a local shared address to the same offset in CTA `rank` of the cluster.
BRI_DEVI uint32_t dsmem_addr(const void* local, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(local)), "r"(rank));
  return out;
}

// (value, index) argmax with LAPACK idamax tie-breaking (first index wins);
// NaN never beats a number (|x| > best is false for NaN).
BRI_DEVI void argmax_merge(double& v, int& i, double ov, int oi) {
  if (ov > v || (ov == v && oi < i)) {
    v = ov;
    i = oi;
  }
}

BRI_DEVI void warp_argmax(double& v, int& i) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, v, off);
    int oi = __shfl_xor_sync(0xffffffffu, i, off);
    argmax_merge(v, i, ov, oi);
  }
}

// Warp-wide argmax of non-negative values with LAPACK idamax tie-breaking
// (smallest index wins).  Lanes with v < 0 (no candidate) or NaN never win;
// if no lane has a candidate the result is (-1, INT_MAX).  Three REDUX
// reductions instead of five shuffle rounds.
BRI_DEVI void warp_argmax_fast(double& v, int& i) {
  const bool ok = (v >= 0.0);
  const unsigned long long bits = ok ? (unsigned long long)__double_as_longlong(v) : 0ull;
  const unsigned hi = (unsigned)(bits >> 32), lo = (unsigned)bits;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  const bool best = ok && hi == mhi && lo == mlo;
  const int mi = (int)__reduce_min_sync(0xffffffffu, best ? (unsigned)i : 0x7fffffffu);
  i = mi;
  v = (mi == 0x7fffffff) ? -1.0 : __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
}

// Value held by the lowest lane whose `owner` flag is set (0.0 if none): used
// to carry a payload (e.g. the signed pivot) alongside warp_argmax_fast.
BRI_DEVI double warp_pick(double v, bool owner) {
  const unsigned m = __ballot_sync(0xffffffffu, owner);
  return m ? __shfl_sync(0xffffffffu, v, __ffs(m) - 1) : 0.0;
}

// Bulk copy of `bytes` (multiple of 16) from this CTA's shared memory into a
// peer CTA's shared memory, completing `bytes` on the peer's mbarrier.
BRI_DEVI void bulk_s2cluster(uint32_t dst_cluster, const void* src, uint32_t bytes, uint32_t mbar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst_cluster),
      "r"(smem_u32(src)), "r"(bytes), "r"(mbar_cluster)
      : "memory");
}

BRI_DEVI void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

BRI_DEVI void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAITC_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

BRI_DEVI double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

BRI_DEVI void lds_f64x2(uint32_t addr, double& a, double& b) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "r"(addr));
}

BRI_DEVI void sts_f64x2(double* p, double a, double b) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(smem_u32(p)), "d"(a), "d"(b) : "memory");
}

}  // namespace bri
