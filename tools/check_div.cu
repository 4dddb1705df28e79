// Checks the quotient used by dinv_kernel (trsm.cu): q = w * r, q1 = fma(fma(-t, q, w), r, q) with
// r = RN(1 / t) against the IEEE division w / t on random operands (normal range, mixed exponents).
// Build + run:  nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/check_div.cu -o /tmp/check_div && /tmp/check_div
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long splitmix(unsigned long long& s) {
  unsigned long long z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ double rnd(unsigned long long& s, int spread) {
  const unsigned long long m = splitmix(s) >> 12;                       // 52 mantissa bits
  const long long e = 1023 + (long long)(splitmix(s) % (2 * spread + 1)) - spread;
  const unsigned long long sign = splitmix(s) & 0x8000000000000000ull;
  return __longlong_as_double((long long)(sign | ((unsigned long long)e << 52) | m));
}
__global__ void check(unsigned long long* bad, unsigned long long* total, int iters, int spread) {
  unsigned long long s = 0x1234567ull * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  unsigned long long nb = 0;
  for (int i = 0; i < iters; ++i) {
    const double w = rnd(s, spread), t = rnd(s, spread);
    const double r = 1.0 / t;
    const double q = w * r;
    const double q1 = fma(fma(-t, q, w), r, q);
    if (__double_as_longlong(q1) != __double_as_longlong(w / t)) ++nb;
  }
  atomicAdd(bad, nb);
  atomicAdd(total, (unsigned long long)iters);
}
int main() {
  unsigned long long *d, h[2];
  cudaMalloc(&d, 16);
  for (int spread : {0, 8, 300}) {
    cudaMemset(d, 0, 16);
    check<<<592, 256>>>(d, d + 1, 20000, spread);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("exponent spread +-%d: %llu of %llu quotients differ from IEEE division (%s)\n", spread, h[0], h[1],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
