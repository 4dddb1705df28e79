// Per-launch time and phase split (clock64, CTA 0) of the one-CTA small-node kernel:
// order n, `items` nodes (config 1's levels are 36 / 64 / 16 nodes), mode 0 (Schur node) and
// mode 1 (inverse), for both schedules (blocked panels per warp / column-cyclic), plus a
// bitwise comparison of their outputs on a diagonally dominant and on a heavily pivoting input.
// Build: see tools/bench_small.sh.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1612_00001_b200/csrc/bri_internal.h"
namespace bri { void small_profile_read(unsigned long long* out); void small_set_blocked(int on); void count_launch() {} }
using namespace bri;
int main(int argc, char** argv) {
  configure_small();
  const int n = argc > 1 ? atoi(argv[1]) : 64, items = argc > 2 ? atoi(argv[2]) : 64, per = 5;
  ArenaView a; a.n = n; a.ld = (n + 7) / 8 * 8; a.slot_elems = (long long)n * a.ld; a.nslots = items * per;
  cudaMalloc(&a.base, sizeof(double) * a.slot_elems * a.nslots);
  std::vector<int> it(items * 5);
  for (int q = 0; q < items; ++q) for (int k = 0; k < 5; ++k) it[q * 5 + k] = q * per + k;
  int* d_it; cudaMalloc(&d_it, it.size() * 4); cudaMemcpy(d_it, it.data(), it.size() * 4, cudaMemcpyHostToDevice);
  int* st; cudaMalloc(&st, items * 4);
  unsigned long long ph[8];
  for (int shift = 1; shift >= 0; --shift) {
    std::vector<double> h(a.slot_elems * a.nslots);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)((i * 2654435761u) % 1000) / 1000.0 - 0.5;
    if (shift)
      for (int s = 0; s < a.nslots; s += per)
        for (int i = 0; i < n; ++i) h[(size_t)s * a.slot_elems + i * a.ld + i] += n;
    for (int mode = 0; mode < 2; ++mode) {
      std::vector<double> out[2];
      std::vector<int> sth[2];
      for (int blk = 0; blk < 2; ++blk) {
        small_set_blocked(blk);
        cudaMemcpy(a.base, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
        cudaMemset(st, 0xff, items * 4);
        launch_small_node(a, d_it, items, mode, st, 0); cudaDeviceSynchronize(); small_profile_read(ph);
        out[blk].resize(h.size()); sth[blk].resize(items);
        cudaMemcpy(out[blk].data(), a.base, sizeof(double) * h.size(), cudaMemcpyDeviceToHost);
        cudaMemcpy(sth[blk].data(), st, items * 4, cudaMemcpyDeviceToHost);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        for (int r = 0; r < 10; ++r) launch_small_node(a, d_it, items, mode, st, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        small_profile_read(ph);
        const char* nm[6] = {"load", "lu+fwd", "bwd", "W+status", "wait_rt", "gemm"};
        printf("n=%d items=%d mode=%d %s %s per launch %.1f us;", n, items, mode, shift ? "dominant" : "pivoting",
               blk ? "blocked" : "cyclic ", ms * 100);
        for (int k = 0; k < 6; ++k) printf(" %s=%.0f", nm[k], ph[k] / 10.0);
        printf(" cyc (%s)\n", cudaGetErrorString(cudaGetLastError()));
      }
      const bool same = memcmp(out[0].data(), out[1].data(), sizeof(double) * h.size()) == 0 &&
                        memcmp(sth[0].data(), sth[1].data(), items * 4) == 0;
      int bad = 0;
      for (int q = 0; q < items; ++q) bad += sth[1][q] != 0;
      printf("  -> blocked vs cyclic outputs and statuses: %s (%d nonzero statuses)\n", same ? "BIT-IDENTICAL" : "DIFFER", bad);
    }
  }
  return 0;
}
