// FP64 pipe probe: DFMA latency (one dependent chain) and throughput (8 independent chains per thread).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, int iters, long long* cyc) {
  double a = out[threadIdx.x], b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); }
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void thr(double* out, int iters, long long* cyc) {
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = out[threadIdx.x] + k;
  const double b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  long long t1 = clock64();
  double s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* out; long long* cyc; long long h;
  cudaMalloc(&out, 1024 * 8); cudaMemset(out, 0, 8192); cudaMalloc(&cyc, 8 * 148);
  const int it = 4096;
  lat<<<1, 32>>>(out, it, cyc); cudaDeviceSynchronize();
  lat<<<1, 32>>>(out, it, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)h / (4.0 * it));
  for (int th : {128, 256, 512, 1024}) {
    thr<<<148, th>>>(out, it, cyc); cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); thr<<<148, th>>>(out, it, cyc); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    double fmas = 148.0 * th * it * 8;
    printf("threads/SM %4d: %.1f DFMA/clk/SM (clock64), %.2f TFLOP/s fp64 (events)\n", th, (double)th * it * 8 / h,
           2 * fmas / ms / 1e9);
  }
  return 0;
}
