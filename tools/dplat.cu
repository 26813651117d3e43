// fp64 dependent-chain latency and LDS/LDTM-like costs on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain_mul(double* out, double a, int n, long long* cyc) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x * a; x = x * a; x = x * a; x = x * a; }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void chain_add(double* out, double a, int n, long long* cyc) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x + a; x = x + a; x = x + a; x = x + a; }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void chain_thomas(double* out, const double* tab, int n, long long* cyc) {
  __shared__ double s[128 * 32];
  __shared__ double tv[129], ti[128];
  for (int k = threadIdx.x; k < 128; k += 32) { ti[k] = tab[k]; tv[k] = tab[k] * 0.5; }
  for (int k = 0; k < 128; ++k) s[k * 32 + threadIdx.x] = out[threadIdx.x] + k;
  __syncwarp();
  double cv = 0.3, g = 1.0;
  long long t0 = clock64();
  for (int r = 0; r < n; ++r) {
#pragma unroll 8
    for (int k = 1; k < 128; ++k) {
      double t = g * cv; t = t * tv[k]; g = s[k * 32 + threadIdx.x] + t; g = g * ti[k];
      s[k * 32 + threadIdx.x] = g;
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = g; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double *o, *tab; long long *c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&tab, 256 * 8); cudaMalloc(&c, 8);
  cudaMemset(o, 0, 1024 * 8); cudaMemset(tab, 0, 256 * 8);
  long long h; int n = 10000;
  chain_mul<<<1, 32>>>(o, 1.0000001, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DMUL dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
  chain_add<<<1, 32>>>(o, 1e-9, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
  chain_thomas<<<1, 32>>>(o, tab, 100, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("Thomas forward step (smem): %.2f cycles/step\n", (double)h / (100.0 * 127));
  // 8 concurrent warps on one SM
  chain_thomas<<<1, 32>>>(o, tab, 100, c);
  return 0;
}
