// Per-launch time and phase split (clock64, CTA 0) of the one-CTA small-node kernel:
// b = 64, `items` nodes (config 1's levels are 36 / 64 / 16 nodes), mode 0 (Schur node)
// and mode 1 (inverse).  Build: see tools/bench_small.sh.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1612_00001_b200/csrc/bri_internal.h"
namespace bri { void small_profile_read(unsigned long long* out); void count_launch() {} }
using namespace bri;
int main(int argc, char** argv) {
  configure_small();
  const int n = argc > 1 ? atoi(argv[1]) : 64, items = argc > 2 ? atoi(argv[2]) : 64, per = 5;
  ArenaView a; a.n = n; a.ld = (n + 7) / 8 * 8; a.slot_elems = (long long)n * a.ld; a.nslots = items * per;
  cudaMalloc(&a.base, sizeof(double) * a.slot_elems * a.nslots);
  std::vector<double> h(a.slot_elems * a.nslots);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)((i * 2654435761u) % 1000) / 1000.0 - 0.5;
  for (int s = 0; s < a.nslots; s += per)
    for (int i = 0; i < n; ++i) h[(size_t)s * a.slot_elems + i * a.ld + i] += n;
  cudaMemcpy(a.base, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
  std::vector<int> it(items * 5);
  for (int q = 0; q < items; ++q) for (int k = 0; k < 5; ++k) it[q * 5 + k] = q * per + k;
  int* d_it; cudaMalloc(&d_it, it.size() * 4); cudaMemcpy(d_it, it.data(), it.size() * 4, cudaMemcpyHostToDevice);
  int* st; cudaMalloc(&st, items * 4);
  unsigned long long ph[8];
  for (int mode = 0; mode < 2; ++mode) {
    launch_small_node(a, d_it, items, mode, st, 0); cudaDeviceSynchronize(); small_profile_read(ph);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) launch_small_node(a, d_it, items, mode, st, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    small_profile_read(ph);
    const char* nm[6] = {"load", "lu+fwd", "bwd", "W+status", "wait_rt", "gemm"};
    printf("n=%d items=%d mode=%d per launch %.1f us;", n, items, mode, ms * 100);
    for (int k = 0; k < 6; ++k) printf(" %s=%.0f", nm[k], ph[k] / 10.0);
    printf(" cyc (%s)\n", cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
