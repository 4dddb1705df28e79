// Microbenchmark of the LU panel kernel alone: time vs panel height and width.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1612_00001_b200/csrc/bri_internal.h"
namespace bri { void count_launch() {} }
using namespace bri;
int main(int argc, char** argv) {
  configure_lu();
  const int n = argc > 1 ? atoi(argv[1]) : 4096;
  ArenaView a;
  a.n = n; a.ld = n; a.slot_elems = (long long)n * n; a.nslots = 1;
  cudaMalloc(&a.base, sizeof(double) * a.slot_elems);
  std::vector<double> h(a.slot_elems);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)((i * 2654435761u) % 1000) / 1000.0 - 0.5;
  cudaMemcpy(a.base, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
  int* slots; cudaMalloc(&slots, 4); cudaMemset(slots, 0, 4);
  LuScratch sc;
  cudaMalloc(&sc.ipiv, n * 4); cudaMalloc(&sc.pi, n * 4); cudaMalloc(&sc.sigma, n * 4);
  cudaMalloc(&sc.pairs, 2000 * 65 * 4); cudaMemset(sc.pairs, 0, 2000 * 65 * 4); cudaMalloc(&sc.orig, n * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int j0 : {0, n / 2, n - 512, n - 256, n - 96}) {
    for (int nb : {1, 4, 16, 32}) {
      for (int w = 0; w < 2; ++w) launch_panel(a, slots, 1, j0, nb, 0, sc, n, 65, 0);
      cudaEventRecord(e0);
      const int reps = 10;
      for (int r = 0; r < reps; ++r) launch_panel(a, slots, 1, j0, nb, 0, sc, n, 65, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("H=%d nb=%d: %.1f us/panel  %.2f us/col  err=%s\n", n - j0, nb, ms * 1000 / reps, ms * 1000 / reps / nb,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
