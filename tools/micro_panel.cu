// Latency microbenchmarks of the LU panel's per-column primitives (dependent chains, clock64).
#include <cstdio>
#include <climits>
#include <cuda_runtime.h>
#include "../paper_1612_00001_b200/csrc/bri_common.cuh"
using namespace bri;

__global__ void k_argmax(long long* out, double seed, int iters) {
  double v = seed + threadIdx.x * 1e-3;
  int i = threadIdx.x;
  const long long t0 = clock64();
  for (int k = 0; k < iters; ++k) {
    double w = v; int j = i;
    warp_argmax_fast(w, j);
    v = w * 0.999 + 1e-9 * j;   // dependent
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / iters; out[1] = (long long)v; }
}

__global__ void k_bar(long long* out, int iters) {
  __shared__ double s[256];
  double v = threadIdx.x;
  const long long t0 = clock64();
  for (int k = 0; k < iters; ++k) {
    s[threadIdx.x] = v;
    __syncthreads();
    v = s[(threadIdx.x + 1) & 255] + 1.0;
    __syncthreads();
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / iters / 2; out[1] = (long long)v; }
}

__global__ void k_div(long long* out, double seed, int iters) {
  double v = seed + threadIdx.x;
  const long long t0 = clock64();
  for (int k = 0; k < iters; ++k) v = 1.0 / (v + 1.5);
  const long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / iters; out[1] = (long long)(v * 1e6); }
}

struct __align__(16) Msg { double d[36]; };

// cluster exchange round: every CTA bulk-copies a 288-byte message to every CTA, waits on its mbarrier
__global__ void k_xchg(long long* out, int iters) {
  __shared__ Msg inbox[2][16];
  __shared__ Msg stg;
  __shared__ __align__(8) uint64_t bar[2];
  const int cs = (int)cluster_nctarank(), rank = (int)cluster_ctarank();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_barrier_init(); }
  for (int e = threadIdx.x; e < 36; e += blockDim.x) stg.d[e] = e;
  cluster_sync_all();
  const long long t0 = clock64();
  for (int k = 0; k < iters; ++k) {
    const int par = k & 1;
    if (threadIdx.x == 0) mbar_arrive_expect_tx(&bar[par], cs * (uint32_t)sizeof(Msg));
    if (warp == 0) {
      fence_proxy_async_smem();
      __syncwarp();
      if (lane < cs) bulk_s2cluster(dsmem_addr(&inbox[par][rank], lane), &stg, sizeof(Msg), dsmem_addr(&bar[par], lane));
    }
    mbar_wait_cluster(&bar[par], (k >> 1) & 1);
    __syncthreads();
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) out[0] = (t1 - t0) / iters;
  cluster_sync_all();
}

int main() {
  long long* d; cudaMalloc(&d, 64); long long h[2];
  k_argmax<<<1, 256>>>(d, 1.0, 1000); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("warp_argmax_fast: %lld cycles\n", h[0]);
  k_bar<<<1, 256>>>(d, 1000); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("sts+syncthreads+lds (256 thr): %lld cycles\n", h[0]);
  k_div<<<1, 32>>>(d, 1.0, 1000); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("dp 1/x: %lld cycles\n", h[0]);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(cs); cfg.blockDim = dim3(256);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1; cfg.attrs = at; cfg.numAttrs = 1;
    if (cs == 16) cudaFuncSetAttribute(k_xchg, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_xchg, d, 1000);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("cluster exchange cs=%d: %lld cycles (%s)\n", cs, h[0], cudaGetErrorString(e));
  }
  return 0;
}
