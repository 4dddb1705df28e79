#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1612_00001_b200/csrc/bri_internal.h"
namespace bri { void panel_profile_read(unsigned long long* out); void count_launch() {} }
using namespace bri;
int main() {
  configure_lu();
  const int n = 4096;
  ArenaView a; a.n = n; a.ld = n; a.slot_elems = (long long)n * n; a.nslots = 1;
  cudaMalloc(&a.base, sizeof(double) * a.slot_elems);
  std::vector<double> h(a.slot_elems);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)((i * 2654435761u) % 1000) / 1000.0 - 0.5;
  cudaMemcpy(a.base, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
  int* slots; cudaMalloc(&slots, 4); cudaMemset(slots, 0, 4);
  LuScratch sc;
  cudaMalloc(&sc.ipiv, n * 4); cudaMalloc(&sc.pi, n * 4); cudaMalloc(&sc.sigma, n * 4);
  cudaMalloc(&sc.pairs, 200 * 65 * 4); cudaMemset(sc.pairs, 0, 200 * 65 * 4);
  unsigned long long ph[10];
  for (int j0 : {0, 1024, 2048, 3072, 3840, 4000}) {
    launch_panel(a, slots, 1, j0, 32, 0, sc, n, 65, 0);
    cudaDeviceSynchronize();
    panel_profile_read(ph);
    for (int r = 0; r < 10; ++r) launch_panel(a, slots, 1, j0, 32, 0, sc, n, 65, 0);
    cudaDeviceSynchronize();
    panel_profile_read(ph);
    printf("H=%d cycles/col:", n - j0);
    const char* nm[9] = {"ctawinner", "bulkissue", "wait", "select", "swap", "update+nextcand", "stage_j", "fence", "stage_cand"};
    for (int k = 0; k < 9; ++k) printf(" %s=%.0f", nm[k], ph[k] / 320.0);
    printf("  err=%s\n", cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
