// FP64 pipe microbenchmark for sm_100a: DMMA (mma.sync f64 shapes) and DFMA.
// Register-only loops with independent accumulator chains; reports TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void k_m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void k_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + threadIdx.x * 1e-4 + i;
  double c[CHAINS][4];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void k_m16n8k4(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-4;
  double c[CHAINS][4];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void k_dfma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - 1e-9;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

template <typename F>
double timeit(F launch, double flops) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return flops / (best * 1e-3) / 1e12;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  double* out; cudaMalloc(&out, 8);
  const int iters = 4096;
  printf("{\"gpu\": \"%s\", \"sms\": %d", p.name, sms);
  for (int warps : {4, 8, 16}) {
    int threads = 32 * warps;
    int blocks = sms * 2;
    double nw = (double)blocks * warps;
    double t1 = timeit([&] { k_m8n8k4<8><<<blocks, threads>>>(out, iters); }, nw * iters * 8 * 2.0 * 8 * 8 * 4);
    double t2 = timeit([&] { k_m16n8k16<4><<<blocks, threads>>>(out, iters / 4); }, nw * (iters / 4) * 4 * 2.0 * 16 * 8 * 16);
    double t3 = timeit([&] { k_m16n8k4<4><<<blocks, threads>>>(out, iters); }, nw * iters * 4 * 2.0 * 16 * 8 * 4);
    double t4 = timeit([&] { k_dfma<8><<<blocks, threads>>>(out, iters); }, nw * 32 * iters * 8 * 2.0);
    printf(", \"w%d\": {\"m8n8k4\": %.2f, \"m16n8k16\": %.2f, \"m16n8k4\": %.2f, \"dfma\": %.2f}", warps, t1, t2, t3, t4);
  }
  printf("}\n");
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
  return 0;
}
