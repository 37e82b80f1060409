// Micro-benchmark (diagnostics): FP64 latency / throughput of the scalar ops
// the small dense kernels chain (DFMA, shuffles, div, sqrt, rsqrt, LDS).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, int n, double x0) {
  double x = x0 + threadIdx.x * 1e-9, y = 1.0000001;
  __shared__ double sh[1024];
  sh[threadIdx.x] = x;
  __syncthreads();
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-12);
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = t1 - t0;
  // shfl chain (double)
  t0 = clock64();
  for (int i = 0; i < n; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = t1 - t0;
  // div chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.5);
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = t1 - t0;
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 1.5);
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = t1 - t0;
  // rsqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x + 1.5);
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = t1 - t0;
  // hypot chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = hypot(x, 0.75);
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = t1 - t0;
  // LDS dependent chain
  int idx = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { double v = sh[idx]; idx = ((int)v & 1) ^ threadIdx.x; x += v; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[6] = t1 - t0;
  // barrier chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64(); if (threadIdx.x == 0) cyc[7] = t1 - t0;
  out[threadIdx.x] = x;
}
// throughput: 8 independent FMA chains per thread, all threads
__global__ void thr(double* out, long long* cyc, int n) {
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x + k;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], 1.0000001, 1e-9);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  double s = 0; for (int k = 0; k < 8; ++k) s += a[k];
  out[threadIdx.x] = s;
}
__global__ void dmma_k(double* out, long long* cyc, int n, int chains) {
  double c[8][2];
  for (int k = 0; k < 8; ++k) { c[k][0] = threadIdx.x; c[k][1] = k; }
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.5;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k < chains)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  double s = 0; for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  out[threadIdx.x] = s;
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 1 << 20); cudaMalloc(&c, 1024);
  const int n = 1000;
  lat<<<1, 32>>>(d, c, n, 0.5); cudaDeviceSynchronize();
  lat<<<1, 32>>>(d, c, n, 0.5);
  long long h[8]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
  const char* nm[8] = {"dfma", "shfl+dadd", "div", "sqrt", "rsqrt", "hypot", "lds", "bar(1warp)"};
  for (int i = 0; i < 8; ++i) printf("latency %-10s %.1f cyc\n", nm[i], (double)h[i] / n);
  for (int t : {32, 128, 256, 512, 1024}) {
    thr<<<1, t>>>(d, c, n); cudaDeviceSynchronize();
    thr<<<1, t>>>(d, c, n);
    cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    printf("throughput threads=%4d: %.2f DFMA/clk/SM\n", t, 8.0 * n * t / h[0]);
  }
  for (int ch : {1, 2, 4, 8})
    for (int t : {32, 128, 512}) {
      dmma_k<<<1, t>>>(d, c, n, ch); cudaDeviceSynchronize();
      dmma_k<<<1, t>>>(d, c, n, ch);
      cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
      printf("dmma chains=%d threads=%4d: %.1f cyc per step (%d dmma/warp/step), %.2f dmma/clk/SM\n", ch, t,
             (double)h[0] / n, ch, (double)ch * n * (t / 32) / h[0]);
    }
  lat<<<1, 512>>>(d, c, n, 0.5); cudaDeviceSynchronize();
  cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
  printf("bar latency with 16 warps: %.1f cyc\n", (double)h[7] / n);
  return 0;
}
